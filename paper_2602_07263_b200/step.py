"""ctypes view of the C++ layer-set training step executor (tlora_step_*, include/tlora.h).

The executor (csrc/tlora_step.cu) is the product path of a training step: rank-aware
nano-batch map, chained fused-GEMM schedule on the caller's stream, side-stream dB+dA
and AdamW, optional data-parallel gradient all-reduce through the C-ABI communicator,
CUDA-graph replay, AIMD on the measured step time (sim_engine.hpp:306-315 executed for
real). This module only builds the descriptor, fills weights / inputs through torch
(device memory plumbing) and reads results back; it schedules nothing itself.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import capi
from .capi import call
from .layer import _CudaArray, _stream_ptr
from .workload import INPUT_GROUP, Workload


@dataclass
class StepStats:
    nano_used: int
    next_nano: int
    ms: float
    replayed_graph: bool
    launches: int
    tokens: int


class _LayerView:
    """The executor-owned tlora_layer of one (layer, projection) key, with the calls the
    drivers need (weights, optimizer, gradients) — same semantics as FusedLoRALayer."""

    def __init__(self, h, d, k, ranks, device):
        self._h, self.d, self.k, self.ranks, self.device = h, d, k, list(ranks), device
        offs = (C.c_int32 * len(self.ranks))()
        R = C.c_int32()
        call("tlora_layer_layout", h, offs, C.byref(R))
        self.offsets, self.R = list(offs), R.value

    def set_base(self, W, stream=None):
        W = W.contiguous()
        call("tlora_layer_set_base", self._h, C.c_void_p(W.data_ptr()), _dt(W), capi.DEVICE,
             _stream_ptr(stream))

    def set_adapter(self, slot, A, B, stream=None):
        A, B = A.contiguous(), B.contiguous()
        call("tlora_layer_set_adapter", self._h, int(slot), C.c_void_p(A.data_ptr()),
             C.c_void_p(B.data_ptr()), _dt(A), capi.DEVICE, _stream_ptr(stream))

    def set_optimizer(self, lr, weight_decay=None, beta1=0.9, beta2=0.999, eps=1e-8):
        S = len(self.ranks)
        lr = [float(lr)] * S if np.isscalar(lr) else [float(x) for x in lr]
        wd = [0.0] * S if weight_decay is None else (
            [float(weight_decay)] * S if np.isscalar(weight_decay) else [float(x) for x in weight_decay])
        call("tlora_layer_set_optimizer", self._h, (C.c_float * S)(*lr), (C.c_float * S)(*wd),
             float(beta1), float(beta2), float(eps))

    def packed_grads(self):
        a, b = C.c_void_p(), C.c_void_p()
        call("tlora_layer_grad_ptrs", self._h, C.byref(a), C.byref(b))
        dev = torch.device("cuda", self.device)
        return (torch.as_tensor(_CudaArray(a.value, (self.R, self.d), "<f4"), device=dev),
                torch.as_tensor(_CudaArray(b.value, (self.R, self.k), "<f4"), device=dev))

    def read_grad(self, slot, stream=None):
        r = self.ranks[slot]
        dev = torch.device("cuda", self.device)
        dA = torch.empty(self.d, r, dtype=torch.float32, device=dev)
        dB = torch.empty(r, self.k, dtype=torch.float32, device=dev)
        call("tlora_layer_read_grad", self._h, int(slot), C.c_void_p(dA.data_ptr()),
             C.c_void_p(dB.data_ptr()), capi.DEVICE, _stream_ptr(stream))
        return dA, dB

    def read_adapter(self, slot, stream=None):
        r = self.ranks[slot]
        dev = torch.device("cuda", self.device)
        A = torch.empty(self.d, r, dtype=torch.float32, device=dev)
        B = torch.empty(r, self.k, dtype=torch.float32, device=dev)
        call("tlora_layer_read_adapter", self._h, int(slot), C.c_void_p(A.data_ptr()),
             C.c_void_p(B.data_ptr()), capi.DEVICE, _stream_ptr(stream))
        return A, B


def _dt(t):
    return {torch.float64: capi.F64, torch.float32: capi.F32, torch.bfloat16: capi.BF16}[t.dtype]


def _torch_view(ptr, rows, cols, dtype, device):
    if dtype == torch.bfloat16:  # no bf16 typestr in the array interface: view int16 bits
        t = torch.as_tensor(_CudaArray(ptr, (rows, cols), "<i2"), device=device)
        return t.view(torch.bfloat16)
    return torch.as_tensor(_CudaArray(ptr, (rows, cols), "<f4"), device=device)


class TrainingStep:
    """One C++ tlora_step over a Workload's layer set.

    nano_fixed > 0 pins N (the reference's config.fixed_n); 0 lets AIMD choose N every
    step from the measured step time, starting at nano_init (reference default 4)."""

    def __init__(self, wl: Workload, device: int = 0, nano_fixed: int = 1, nano_init: int = 4,
                 side_grads: bool = True, graphs: bool = True, dh_ring: int = 8,
                 input_sets: int = 1, comm=None, y_dtype=torch.bfloat16, aimd_alpha: int = 4,
                 aimd_beta: float = 0.5, aimd_tau_rel: float = 0.0, early_grads: bool | None = None,
                 sharded_opt: bool = False):
        self.wl, self.device = wl, int(device)
        self.dev = torch.device("cuda", self.device)
        self.names = [p[0] for p in wl.projections]
        groups = []
        for name in self.names:
            g = INPUT_GROUP.get(name, name)
            if g not in groups:
                groups.append(g)
        self.groups = groups
        P, S = len(wl.projections), len(wl.jobs)
        self._arrs = dict(
            d=(C.c_int64 * P)(*[p[1] for p in wl.projections]),
            k=(C.c_int64 * P)(*[p[2] for p in wl.projections]),
            inp=(C.c_int32 * P)(*[groups.index(INPUT_GROUP.get(n, n)) for n in self.names]),
            ranks=(C.c_int32 * S)(*[j.rank for j in wl.jobs]),
            batch=(C.c_int32 * S)(*[j.batch for j in wl.jobs]),
            seq=(C.c_int32 * S)(*[j.seq_len for j in wl.jobs]))
        a = self._arrs
        if early_grads is None:  # A/B knob
            import os
            early_grads = os.environ.get("TLORA_EARLY_GRADS", "0") == "1"
        flags = ((capi.STEP_SIDE_GRADS if side_grads else 0) | (capi.STEP_GRAPH if graphs else 0)
                 | (capi.STEP_EARLY_GRADS if early_grads and side_grads else 0)
                 | (capi.STEP_SHARDED_OPT if sharded_opt else 0))
        desc = capi.StepDescC(self.device, wl.layers, P, a["d"], a["k"], a["inp"], S, a["ranks"],
                              a["batch"], a["seq"], capi.BF16 if y_dtype == torch.bfloat16 else capi.F32,
                              flags, dh_ring, input_sets, nano_init, nano_fixed, aimd_alpha,
                              aimd_beta, aimd_tau_rel)
        h = C.c_void_p()
        call("tlora_step_create", C.byref(desc), comm, C.byref(h))
        self._h = h
        self.input_sets = input_sets
        self.y_dtype = y_dtype
        self.layers = {}
        for L in range(wl.layers):
            for p, (name, d, k) in enumerate(wl.projections):
                lh = C.c_void_p()
                call("tlora_step_layer", self._h, L, p, C.byref(lh))
                self.layers[(L, name)] = _LayerView(lh, d, k, wl.ranks, self.device)
        self.keys = list(self.layers)
        self.R = self.layers[self.keys[0]].R
        self.T = wl.tokens
        self.X = [{g: self._buf(capi.BUF_X, i, s, torch.bfloat16) for i, g in enumerate(groups)}
                  for s in range(input_sets)]
        self.dY = [{n: self._buf(capi.BUF_DY, p, s, torch.bfloat16) for p, n in enumerate(self.names)}
                   for s in range(input_sets)]
        self.Y = {n: self._buf(capi.BUF_Y, p, 0, y_dtype) for p, n in enumerate(self.names)}
        self.dX = {n: self._buf(capi.BUF_DX, p, 0, torch.bfloat16) for p, n in enumerate(self.names)}
        self.H = {key: self._buf(capi.BUF_H, i, 0, torch.bfloat16) for i, key in enumerate(self.keys)}
        self.trajectory = []

    def _buf(self, kind, index, s, dtype):
        p, r, c = C.c_void_p(), C.c_int64(), C.c_int64()
        call("tlora_step_buffer", self._h, kind, index, s, C.byref(p), C.byref(r), C.byref(c))
        return _torch_view(p.value, r.value, c.value, dtype, self.dev)

    # ---- initialisation: the same values, in the same generator order, as
    # runner.LayerSetStep(wl, seed=seed) (so the two drivers can be compared bit for bit)
    def init_random(self, seed: int | None = None, keep_weights: bool = False):
        wl, dev = self.wl, self.dev
        g = torch.Generator(device=dev)
        g.manual_seed(wl.seed if seed is None else seed)
        T = self.T
        self.weights = {} if keep_weights else None
        seen_g, seen_p = set(), set()
        dims = {name: (d, k) for name, d, k in wl.projections}
        for key in self.keys:
            L, name = key
            d, k = dims[name]
            lay = self.layers[key]
            W = torch.randn(d, k, generator=g, device=dev, dtype=torch.float32).mul_(d ** -0.5)
            W = W.bfloat16()
            lay.set_base(W)
            ab = []
            for s, j in enumerate(wl.jobs):
                A = torch.randn(d, j.rank, generator=g, device=dev).mul_(d ** -0.5).bfloat16()
                B = torch.randn(j.rank, k, generator=g, device=dev).mul_(j.rank ** -0.5).bfloat16()
                lay.set_adapter(s, A, B)
                ab.append((A, B))
            if keep_weights:
                self.weights[key] = (W, ab)
            grp = INPUT_GROUP.get(name, name)
            if grp not in seen_g:
                seen_g.add(grp)
                self.X[0][grp].copy_(torch.randn(T, d, generator=g, device=dev).bfloat16())
            if name not in seen_p:
                seen_p.add(name)
                self.dY[0][name].copy_(torch.randn(T, k, generator=g, device=dev).bfloat16())
        for s in range(1, self.input_sets):
            for grp in self.groups:
                self.X[s][grp].copy_(self.X[0][grp])
            for name in self.names:
                self.dY[s][name].copy_(self.dY[0][name])
        torch.cuda.synchronize(dev)

    def enable_optimizer(self, base_lr: float = 1e-4, weight_decay: float = 0.01):
        """Per-job AdamW hyperparameters, as runner.LayerSetStep.enable_optimizer."""
        lrs = [base_lr * (1.0 + 0.25 * (s % 4)) for s in range(len(self.wl.jobs))]
        for lay in self.layers.values():
            lay.set_optimizer(lrs, weight_decay)
        self.lrs, self.weight_decay = lrs, weight_decay

    # ---- execution
    def run(self, input_set: int = 0, eager: bool = False, stream=None,
            trace: bool = False) -> StepStats:
        st = capi.StepStatsC()
        flags = (capi.RUN_EAGER if eager else 0) | (capi.RUN_TRACE if trace else 0)
        call("tlora_step_run", self._h, int(input_set), flags, _stream_ptr(stream), C.byref(st))
        s = StepStats(st.nano_used, st.next_nano, st.ms, bool(st.replayed_graph), st.launches,
                      st.tokens)
        self.trajectory.append((s.nano_used, s.ms))
        return s

    def set_controller(self, nano_fixed: int = 0, nano_init: int = 4, alpha: int = 4,
                       beta: float = 0.5, tau_rel: float = 0.0):
        """nano_fixed > 0 pins N; 0 = AIMD from nano_init with a fresh controller state."""
        call("tlora_step_set_controller", self._h, int(nano_fixed), int(nano_init), int(alpha),
             float(beta), float(tau_rel))

    def trace(self):
        """[(op dict, end_ms)] of the last run(trace=True) step, schedule order."""
        n = C.c_int32()
        call("tlora_step_trace", self._h, None, None, 0, C.byref(n))
        ops = (capi.StepOpC * max(1, n.value))()
        ms = (C.c_double * max(1, n.value))()
        call("tlora_step_trace", self._h, ops, ms, n.value, C.byref(n))
        return [({f: getattr(o, f) for f, _ in capi.StepOpC._fields_}, ms[i])
                for i, o in enumerate(ops[: n.value])]

    def next_n(self) -> int:
        n = C.c_int32()
        call("tlora_step_next_n", self._h, C.byref(n))
        return n.value

    def layout(self, n: int):
        """(n_used, nano_t0[n+1], nano_slot[n x S], sample_row[samples]) of nano count n."""
        S = len(self.wl.jobs)
        total = sum(j.batch for j in self.wl.jobs)
        m = max(1, min(n, total))
        t0 = np.zeros(m + 1, np.int64)
        ns = np.zeros(m * S, np.int32)
        sr = np.zeros(total, np.int64)
        out = C.c_int32()
        call("tlora_step_layout", self._h, int(n), C.byref(out), t0.ctypes.data, ns.ctypes.data,
             sr.ctypes.data)
        return out.value, t0, ns.reshape(m, S), sr

    def close(self):
        if getattr(self, "_h", None):
            capi.lib().tlora_step_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def schedule_host(keys: int, nano: int, ring: int = 8, side_grads: bool | int = True,
                  data_parallel: bool | int = False):
    """The executor's op list for (keys, nano-batches) (host-only, no device)."""
    n = C.c_int32()
    call("tlora_step_schedule_host", keys, nano, ring, int(side_grads), int(data_parallel), None, 0,
         C.byref(n))
    buf = (capi.StepOpC * max(1, n.value))()
    call("tlora_step_schedule_host", keys, nano, ring, int(side_grads), int(data_parallel), buf,
         n.value, C.byref(n))
    return [{f: getattr(o, f) for f, _ in capi.StepOpC._fields_} for o in buf[: n.value]]


def nano_assign(batch, weight, n):
    """Rank-aware sample -> nano-batch map (tlora_nano_assign, host-only)."""
    batch = np.ascontiguousarray(batch, np.int32)
    weight = np.ascontiguousarray(weight, np.int64)
    S, total = len(batch), int(batch.sum())
    m = max(1, min(max(n, 1), max(total, 1)))
    per = np.zeros(m, np.int32)
    sn = np.zeros(max(1, total), np.int32)
    ns = np.zeros(m * S, np.int32)
    out = C.c_int32()
    code = capi.lib().tlora_nano_assign(S, batch.ctypes.data, weight.ctypes.data, int(n),
                                        C.byref(out), per.ctypes.data, sn.ctypes.data,
                                        ns.ctypes.data)
    if code == capi.ERR_PLAN:
        raise ValueError(capi.lib().tlora_last_error().decode())
    capi.check(code)
    k = out.value
    return k, per[:k].tolist(), sn[:total], ns[: k * S].reshape(k, S)


def sample_weights(wl: Workload):
    """Per-sample work the executor balances (tlora_step_create): seq_len x (sum_p 2 d k +
    rank x sum_p 3 (d + k)) — half the fwd+bwd FLOPs of one sample, in integers."""
    base = sum(2 * d * k for _, d, k in wl.projections)
    ext = sum(3 * (d + k) for _, d, k in wl.projections)
    return [j.seq_len * (base + ext * j.rank) for j in wl.jobs]
