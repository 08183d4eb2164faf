"""Torch-facing wrapper of the fused multi-LoRA layer (C-ABI in include/tlora.h).

PyTorch is only plumbing here: device memory, streams and the process group. All
arithmetic on the path runs in the sm_100a kernels of libtlora.so.

Reference semantics: proj/include/lora_fleet/fused_lora.hpp:84-119 (forward; backward
is new — the reference has none).
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import capi
from .capi import call


def _stream_ptr(stream) -> C.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _ptr(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


class _CudaArray:
    """Minimal __cuda_array_interface__ view over a device pointer owned by the library."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": typestr, "data": (ptr, False), "version": 3,
            "strides": None,
        }


_DT = {torch.float64: capi.F64, torch.float32: capi.F32, torch.bfloat16: capi.BF16}


@dataclass
class PlanInfo:
    tokens: int
    d: int
    k: int
    num_slots: int
    rank_pad_total: int
    num_tiles: tuple
    splits_db: int
    splits_da: int
    useful_ext_cols: int
    packed_ext_cols: int


class Plan:
    """Rank-aware tile-packing / indexing plan of one (nano-)batch (opaque, immutable)."""

    def __init__(self, layer: "FusedLoRALayer", token_slot: Sequence[int], gathered: bool = False):
        ts = np.ascontiguousarray(np.asarray(token_slot, dtype=np.int32))
        self.layer = layer
        self.tokens = int(ts.shape[0])
        self.token_slot = ts
        self.gathered = bool(gathered)
        h = C.c_void_p()
        call("tlora_plan_create_gathered" if gathered else "tlora_plan_create", layer._h,
             self.tokens, ts.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(h))
        self._h = h

    def row_map(self) -> np.ndarray:
        """Original token of each gathered row (identity for a plain plan)."""
        out = np.empty(self.tokens, np.int32)
        call("tlora_plan_row_map", self._h, out.ctypes.data_as(C.POINTER(C.c_int32)))
        return out

    def gather(self, pairs, stream=None):
        """dst[r] = src[row_map[r]] for (src, dst) bf16 T x w tensors (tlora_gather_rows):
        the gathered-order operands X / dY of a gathered plan."""
        n = len(pairs)
        if n == 0:
            return
        for src, dst in pairs:
            assert src.dtype == torch.bfloat16 and dst.dtype == torch.bfloat16
            assert src.shape == dst.shape and src.shape[0] == self.tokens
            assert src.is_contiguous() and dst.is_contiguous()
        srcs = (C.c_void_p * n)(*[p[0].data_ptr() for p in pairs])
        dsts = (C.c_void_p * n)(*[p[1].data_ptr() for p in pairs])
        widths = (C.c_int64 * n)(*[p[0].shape[1] for p in pairs])
        call("tlora_gather_rows", self._h, n, srcs, dsts, widths, _stream_ptr(stream))

    def present_mask(self) -> int:
        """Device pointer to the plan's per-slot presence flags (int32, num_slots)."""
        p = C.c_void_p()
        call("tlora_plan_present_mask", self._h, C.byref(p))
        return p.value

    def info(self) -> PlanInfo:
        i = capi.PlanInfoC()
        call("tlora_plan_get_info", self._h, C.byref(i))
        return PlanInfo(i.tokens, i.d, i.k, i.num_slots, i.rank_pad_total, tuple(i.num_tiles),
                        i.splits_db, i.splits_da, i.useful_ext_cols, i.packed_ext_cols)

    def tiles(self, launch: int) -> np.ndarray:
        n = C.c_int32()
        call("tlora_plan_get_tiles", self._h, launch, None, 0, C.byref(n))
        buf = (capi.TileC * max(1, n.value))()
        call("tlora_plan_get_tiles", self._h, launch, buf, n.value, C.byref(n))
        arr = np.frombuffer(buf, dtype=np.int32).reshape(-1, 8)[: n.value]
        return arr.copy()

    def device_tiles(self, launch: int):
        """(tile table as uploaded, token slots as uploaded), read back from device memory."""
        n = C.c_int32()
        call("tlora_plan_read_device", self._h, launch, None, 0, C.byref(n), None)
        buf = (capi.TileC * max(1, n.value))()
        slots = np.empty(self.tokens, np.int32)
        call("tlora_plan_read_device", self._h, launch, buf, n.value, C.byref(n),
             slots.ctypes.data)
        return np.frombuffer(buf, dtype=np.int32).reshape(-1, 8)[: n.value].copy(), slots

    def close(self):
        if getattr(self, "_h", None):
            capi.lib().tlora_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class FusedLoRALayer:
    """One adapted projection of the Shared Super-Model: frozen W (d x k) + per-job adapters.

    Slots follow the reference adapter order (std::map by job_id, fused_lora.hpp:48-53).
    """

    def __init__(self, d: int, k: int, ranks: Sequence[int], device: int = 0):
        self.d, self.k, self.device = int(d), int(k), int(device)
        self.ranks = [int(r) for r in ranks]
        rk = (C.c_int32 * len(self.ranks))(*self.ranks)
        h = C.c_void_p()
        call("tlora_layer_create", self.device, self.d, self.k, len(self.ranks), rk, C.byref(h))
        self._h = h
        self._plans = weakref.WeakSet()
        offs = (C.c_int32 * len(self.ranks))()
        R = C.c_int32()
        call("tlora_layer_layout", self._h, offs, C.byref(R))
        self.offsets = list(offs)
        self.R = R.value

    # ---------------------------------------------------------------- registry
    def set_base(self, W: torch.Tensor, stream=None):
        W = W.contiguous()
        assert tuple(W.shape) == (self.d, self.k)
        where = capi.DEVICE if W.is_cuda else capi.HOST
        call("tlora_layer_set_base", self._h, _ptr(W), _DT[W.dtype], where, _stream_ptr(stream))

    def set_adapter(self, slot: int, A: torch.Tensor, B: torch.Tensor, stream=None):
        A, B = A.contiguous(), B.contiguous()
        assert A.dtype == B.dtype and A.is_cuda == B.is_cuda
        where = capi.DEVICE if A.is_cuda else capi.HOST
        call("tlora_layer_set_adapter", self._h, int(slot), _ptr(A), _ptr(B), _DT[A.dtype], where,
             _stream_ptr(stream))

    def zero_grad(self, stream=None):
        call("tlora_layer_zero_grad", self._h, _stream_ptr(stream))

    def packed_grads(self):
        """(dAᵀcat [R x d], dBcat [R x k]) fp32 device tensors aliasing the layer's buffers."""
        a, b = C.c_void_p(), C.c_void_p()
        call("tlora_layer_grad_ptrs", self._h, C.byref(a), C.byref(b))
        dev = torch.device("cuda", self.device)
        dAT = torch.as_tensor(_CudaArray(a.value, (self.R, self.d), "<f4"), device=dev)
        dB = torch.as_tensor(_CudaArray(b.value, (self.R, self.k), "<f4"), device=dev)
        return dAT, dB

    def read_grad(self, slot: int, stream=None):
        r = self.ranks[slot]
        dev = torch.device("cuda", self.device)
        dA = torch.empty(self.d, r, dtype=torch.float32, device=dev)
        dB = torch.empty(r, self.k, dtype=torch.float32, device=dev)
        call("tlora_layer_read_grad", self._h, int(slot), _ptr(dA), _ptr(dB), capi.DEVICE,
             _stream_ptr(stream))
        return dA, dB

    # ---------------------------------------------------------------- optimizer
    def set_optimizer(self, lr, weight_decay=None, beta1=0.9, beta2=0.999, eps=1e-8):
        """Fused multi-job AdamW; lr / weight_decay: scalar or one value per slot."""
        S = len(self.ranks)
        lr = [float(lr)] * S if np.isscalar(lr) else [float(x) for x in lr]
        wd = [0.0] * S if weight_decay is None else (
            [float(weight_decay)] * S if np.isscalar(weight_decay) else [float(x) for x in weight_decay])
        call("tlora_layer_set_optimizer", self._h, (C.c_float * S)(*lr), (C.c_float * S)(*wd),
             float(beta1), float(beta2), float(eps))

    def optimizer_step(self, grad_scale=1.0, stream=None, plan: "Plan | None" = None):
        """plan: only the slots with tokens in that plan's batch take a step (jobs absent
        from the step keep masters, moments and step count); None = every slot."""
        if plan is None:
            call("tlora_layer_optimizer_step", self._h, C.c_float(grad_scale), _stream_ptr(stream))
            return
        call("tlora_layer_optimizer_step_masked", self._h, C.c_void_p(plan.present_mask()),
             C.c_float(grad_scale), _stream_ptr(stream))

    def read_adapter(self, slot: int, stream=None):
        r = self.ranks[slot]
        dev = torch.device("cuda", self.device)
        A = torch.empty(self.d, r, dtype=torch.float32, device=dev)
        B = torch.empty(r, self.k, dtype=torch.float32, device=dev)
        call("tlora_layer_read_adapter", self._h, int(slot), _ptr(A), _ptr(B), capi.DEVICE,
             _stream_ptr(stream))
        return A, B

    # ---------------------------------------------------------------- compute
    def plan(self, token_slot: Sequence[int], gathered: bool = False) -> Plan:
        """gathered=True: tlora_plan_create_gathered (operands in job-sorted order via
        Plan.gather, Y / dX written back in token order by the GEMM epilogues)."""
        p = Plan(self, token_slot, gathered)
        self._plans.add(p)
        return p

    def forward(self, plan: Plan, X: torch.Tensor, Y: torch.Tensor | None = None,
                H: torch.Tensor | None = None, y_dtype=torch.bfloat16, stream=None):
        T = plan.tokens
        assert X.dtype == torch.bfloat16 and X.is_contiguous() and tuple(X.shape) == (T, self.d)
        if Y is None:
            Y = torch.empty(T, self.k, dtype=y_dtype, device=X.device)
        if H is None:
            H = torch.empty(T, self.R, dtype=torch.bfloat16, device=X.device)
        call("tlora_forward", self._h, plan._h, _ptr(X), _ptr(Y), _DT[Y.dtype], _ptr(H),
             _stream_ptr(stream))
        return Y, H

    def backward(self, plan: Plan, dY: torch.Tensor, X: torch.Tensor, H: torch.Tensor,
                 dX: torch.Tensor | None | bool = True, beta: float = 0.0, stream=None):
        T = plan.tokens
        assert dY.dtype == torch.bfloat16 and tuple(dY.shape) == (T, self.k)
        if dX is True:
            dX = torch.empty(T, self.d, dtype=torch.bfloat16, device=dY.device)
        elif dX is False:
            dX = None
        call("tlora_backward", self._h, plan._h, _ptr(dY), _ptr(X), _ptr(H), _ptr(dX),
             C.c_float(beta), _stream_ptr(stream))
        return dX

    # ---- per-launch entry points (tensor-parallel / nano-batch drivers)
    def shrink(self, plan: Plan, X, H, stream=None):
        call("tlora_forward_shrink", self._h, plan._h, _ptr(X), _ptr(H), _stream_ptr(stream))

    def fused_gemm(self, plan: Plan, X, H, Y, stream=None):
        call("tlora_forward_gemm", self._h, plan._h, _ptr(X), _ptr(H), _ptr(Y), _DT[Y.dtype],
             _stream_ptr(stream))

    def fused_gemm_shrink(self, plan: Plan, X, H, Y, nxt: "FusedLoRALayer", next_plan: Plan,
                          X_next, H_next, zero_next=True, stream=None):
        """fused_gemm of this layer + shrink of `nxt` as extra tiles of the same launch
        (tlora_forward_gemm_shrink); bit-identical to fused_gemm then nxt.shrink."""
        call("tlora_forward_gemm_shrink", self._h, plan._h, _ptr(X), _ptr(H), _ptr(Y),
             _DT[Y.dtype], nxt._h, next_plan._h, _ptr(X_next), _ptr(H_next), int(zero_next),
             _stream_ptr(stream))

    def fused_gemm_dh(self, plan: Plan, X, H, Y, nxt: "FusedLoRALayer", next_plan: Plan,
                      dY_next, dH_next, zero_next=True, stream=None):
        """fused_gemm of this layer + dh of `nxt` in one launch (tlora_forward_gemm_dh)."""
        call("tlora_forward_gemm_dh", self._h, plan._h, _ptr(X), _ptr(H), _ptr(Y),
             _DT[Y.dtype], nxt._h, next_plan._h, _ptr(dY_next), _ptr(dH_next), int(zero_next),
             _stream_ptr(stream))

    def fused_gemm_rs(self, plan: Plan, X, H, recv_ptrs, rank, slot_rows, dst_row0, stream=None):
        """Row-parallel TP forward with the reduce-scatter fused into the epilogue (peer
        stores into every owner's receive slot); see tlora_forward_gemm_rs."""
        ptrs = (C.c_void_p * len(recv_ptrs))(*[int(p) for p in recv_ptrs])
        call("tlora_forward_gemm_rs", self._h, plan._h, _ptr(X), _ptr(H), ptrs, len(recv_ptrs),
             int(rank), int(slot_rows), int(dst_row0), _stream_ptr(stream))

    def dh(self, plan: Plan, dY, dH, stream=None):
        call("tlora_backward_dh", self._h, plan._h, _ptr(dY), _ptr(dH), _stream_ptr(stream))

    def dx(self, plan: Plan, dY, dH, dX, beta=0.0, stream=None):
        call("tlora_backward_dx", self._h, plan._h, _ptr(dY), _ptr(dH), _ptr(dX), C.c_float(beta),
             _stream_ptr(stream))

    def dx_dh(self, plan: Plan, dY, dH, dX, nxt: "FusedLoRALayer", next_plan: Plan, dY_next,
              dH_next, beta=0.0, zero_next=True, stream=None):
        """dx of this layer + dh of `nxt` in one launch (tlora_backward_dx_dh)."""
        call("tlora_backward_dx_dh", self._h, plan._h, _ptr(dY), _ptr(dH), _ptr(dX),
             C.c_float(beta), nxt._h, next_plan._h, _ptr(dY_next), _ptr(dH_next),
             int(zero_next), _stream_ptr(stream))

    def grads(self, plan: Plan, H, dY, X, dH, beta=0.0, stream=None):
        """dB and dA in one launch (tlora_backward_grads)."""
        call("tlora_backward_grads", self._h, plan._h, _ptr(H), _ptr(dY), _ptr(X), _ptr(dH),
             C.c_float(beta), _stream_ptr(stream))

    def grad_b(self, plan: Plan, H, dY, beta=0.0, stream=None):
        call("tlora_backward_grad_b", self._h, plan._h, _ptr(H), _ptr(dY), C.c_float(beta),
             _stream_ptr(stream))

    def grad_a(self, plan: Plan, X, dH, beta=0.0, stream=None):
        call("tlora_backward_grad_a", self._h, plan._h, _ptr(X), _ptr(dH), C.c_float(beta),
             _stream_ptr(stream))

    def close(self):
        if getattr(self, "_h", None):
            for p in list(getattr(self, "_plans", ())):
                p.close()
            capi.lib().tlora_layer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def reduce_slots(recv, world, slot_rows, row0, rows, k, out, stream=None):
    call("tlora_reduce_slots", _ptr(recv), int(world), int(slot_rows), int(row0), int(rows),
         int(k), _ptr(out), _stream_ptr(stream))


def grad_schedule_host(d: int, k: int, ranks, token_slot, ctas: int):
    """(off[ctas+1], idx): the LPT CTA tile lists of the plan's dB+dA launch (host only)."""
    rk = (C.c_int32 * len(ranks))(*[int(r) for r in ranks])
    ts = np.ascontiguousarray(np.asarray(token_slot, dtype=np.int32))
    n = C.c_int32()
    off = np.zeros(ctas + 1, np.int32)
    I32 = C.POINTER(C.c_int32)
    call("tlora_plan_grad_schedule_host", int(d), int(k), len(ranks), rk, int(ts.shape[0]),
         ts.ctypes.data_as(I32), int(ctas), off.ctypes.data_as(I32), None, 0, C.byref(n))
    idx = np.zeros(max(1, n.value), np.int32)
    call("tlora_plan_grad_schedule_host", int(d), int(k), len(ranks), rk, int(ts.shape[0]),
         ts.ctypes.data_as(I32), int(ctas), off.ctypes.data_as(I32), idx.ctypes.data_as(I32),
         n.value, C.byref(n))
    return off, idx[: n.value]


def plan_tiles_host(d: int, k: int, ranks, token_slot, launch: int) -> np.ndarray:
    """Host-only tile table (no device), identical to what Plan uploads."""
    rk = (C.c_int32 * len(ranks))(*[int(r) for r in ranks])
    ts = np.ascontiguousarray(np.asarray(token_slot, dtype=np.int32))
    n = C.c_int32()
    call("tlora_plan_tiles_host", int(d), int(k), len(ranks), rk, int(ts.shape[0]),
         ts.ctypes.data_as(C.POINTER(C.c_int32)), int(launch), None, 0, C.byref(n))
    buf = (capi.TileC * max(1, n.value))()
    call("tlora_plan_tiles_host", int(d), int(k), len(ranks), rk, int(ts.shape[0]),
         ts.ctypes.data_as(C.POINTER(C.c_int32)), int(launch), buf, n.value, C.byref(n))
    return np.frombuffer(buf, dtype=np.int32).reshape(-1, 8)[: n.value].copy()


def op_cost(tokens: int, d: int, k: int, tokens_per_slot, ranks, fused: bool = True):
    """Reference OpCost (fused_lora.hpp:95-116 fused, :139-163 unfused), bit-identical."""
    n = len(ranks)
    tp = (C.c_int64 * n)(*[int(x) for x in tokens_per_slot])
    rk = (C.c_int32 * n)(*[int(x) for x in ranks])
    f, b, l = C.c_double(), C.c_double(), C.c_longlong()
    call("tlora_op_cost", int(tokens), int(d), int(k), n, tp, rk, int(bool(fused)), C.byref(f),
         C.byref(b), C.byref(l))
    return f.value, b.value, l.value


def segments(token_slot, num_slots: int):
    """Job-sorted permutation + CSR offsets (tlora_segments; fused_lora.hpp:56-61
    segment_rows for every job at once): perm[offsets[s]:offsets[s+1]] = rows of slot s."""
    slots = np.ascontiguousarray(token_slot, dtype=np.int32)
    perm = np.empty(slots.shape[0], np.int64)
    offsets = np.empty(num_slots + 1, np.int64)
    call("tlora_segments", slots.shape[0], slots.ctypes.data, int(num_slots), perm.ctypes.data,
         offsets.ctypes.data)
    return perm, offsets


def monitor(t_comp, t_comm, t_iter_event: float, t_iter_analytic: float, num_stages: int = 1):
    """nano_pipeline.hpp:114-126 MonitorReading of a PipelineTrace (:28-34): eta_util =
    sum(t_comp) / (num_stages * t_iter_event) (0 if t_iter_event <= 0 or no stages),
    delta_stall = t_iter_event - t_iter_analytic. t_comm is part of the trace but, as in
    the reference, does not enter the reading."""
    sum_c = float(sum(t_comp))
    eta = sum_c / (num_stages * t_iter_event) if t_iter_event > 0.0 and num_stages > 0 else 0.0
    return eta, t_iter_event - t_iter_analytic


def partition(group_batch: int, n: int):
    """nano_pipeline.hpp:51-60 — returns (n, per_nano_samples)."""
    out_n = C.c_int32()
    buf = (C.c_int32 * max(1, min(max(n, 1), max(group_batch, 1))))()
    code = capi.lib().tlora_partition(int(group_batch), int(n), C.byref(out_n), buf)
    if code == capi.ERR_PLAN:
        raise ValueError(capi.lib().tlora_last_error().decode())
    capi.check(code)
    return out_n.value, list(buf)[: out_n.value]


@dataclass
class AimdState:
    """nano_pipeline.hpp:36-47 (defaults n=4, alpha=4, beta=0.5, tau_rel=0)."""
    n: int = 4
    t_prev: float | None = None
    alpha: int = 4
    beta: float = 0.5
    tau_rel: float = 0.0


def aimd_step(state: AimdState, t_t: float) -> AimdState:
    """nano_pipeline.hpp:99-112, via the C-ABI (bit-exact)."""
    n = C.c_int32(state.n)
    hp = C.c_int32(0 if state.t_prev is None else 1)
    tp = C.c_double(0.0 if state.t_prev is None else state.t_prev)
    code = capi.lib().tlora_aimd_step(C.byref(n), C.byref(hp), C.byref(tp), state.alpha,
                                      state.beta, state.tau_rel, float(t_t))
    if code == capi.ERR_PLAN:
        raise ValueError(capi.lib().tlora_last_error().decode())
    capi.check(code)
    return AimdState(n.value, tp.value, state.alpha, state.beta, state.tau_rel)
