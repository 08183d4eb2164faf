"""ctypes view of the C++ tensor-parallel step (tlora_tp_*, csrc/tlora_tp.cu).

Same sharding, nano-batch map, boundary traffic and schedule as the round-1 Python driver
(`tp.TPLayerSetStep`), executed by the library: this module only builds the descriptor,
loads the shards of the full weights (identical seeds and generator order as the Python
driver, so the two can be compared) and reads buffers back.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import capi
from .capi import call
from .layer import _stream_ptr
from .step import StepStats, _LayerView, _torch_view
from .tp import COLUMN, ROW, shard_columns, shard_rows
from .workload import INPUT_GROUP, Workload

TP_FUSED_RS, TP_COPY_ENGINE, TP_SIDE_GRADS = 1, 2, 4
(BUF_X_SHARD, BUF_X_LOC, BUF_DY, BUF_DY_SHARD, BUF_Y, BUF_Y_SHARD, BUF_DX_SHARD,
 BUF_DX_LOC) = range(8)


class TPDescC(C.Structure):
    _fields_ = [
        ("device", C.c_int32), ("num_projections", C.c_int32),
        ("proj_d", C.POINTER(C.c_int64)), ("proj_k", C.POINTER(C.c_int64)),
        ("proj_input", C.POINTER(C.c_int32)), ("proj_row_parallel", C.POINTER(C.c_int32)),
        ("num_slots", C.c_int32), ("ranks", C.POINTER(C.c_int32)),
        ("batch", C.POINTER(C.c_int32)), ("seq_len", C.POINTER(C.c_int32)),
        ("flags", C.c_int32), ("nano_init", C.c_int32), ("nano_fixed", C.c_int32),
        ("aimd_alpha", C.c_int32), ("aimd_beta", C.c_double), ("aimd_tau_rel", C.c_double),
    ]


class TPExecutor:
    def __init__(self, wl: Workload, rank: int, world: int, device: int, comm,
                 nano_fixed: int = 0, nano_init: int = 4, fused_rs: bool = True,
                 copy_engine: bool = True, side_grads: bool = True, seed: int | None = None):
        self.wl, self.rank, self.world = wl, rank, world
        self.dev = torch.device("cuda", device)
        self.device = device
        P = world
        names = [p[0] for p in wl.projections]
        self.names = names
        # input groups of the column-parallel projections, sorted by name (the Python
        # driver's order, so the seeded inputs land in the same buffers)
        self.groups = sorted({INPUT_GROUP[p] for p in COLUMN if p in names})
        NP, S = len(names), len(wl.jobs)
        self._arrs = dict(
            d=(C.c_int64 * NP)(*[p[1] for p in wl.projections]),
            k=(C.c_int64 * NP)(*[p[2] for p in wl.projections]),
            inp=(C.c_int32 * NP)(*[self.groups.index(INPUT_GROUP[n]) if n in COLUMN else 0
                                   for n in names]),
            row=(C.c_int32 * NP)(*[1 if n in ROW else 0 for n in names]),
            ranks=(C.c_int32 * S)(*[j.rank for j in wl.jobs]),
            batch=(C.c_int32 * S)(*[j.batch for j in wl.jobs]),
            seq=(C.c_int32 * S)(*[j.seq_len for j in wl.jobs]))
        a = self._arrs
        flags = ((TP_FUSED_RS if fused_rs else 0) | (TP_COPY_ENGINE if copy_engine else 0)
                 | (TP_SIDE_GRADS if side_grads else 0))
        desc = TPDescC(device, NP, a["d"], a["k"], a["inp"], a["row"], S, a["ranks"], a["batch"],
                       a["seq"], flags, nano_init, nano_fixed, 4, 0.5, 0.0)
        h = C.c_void_p()
        call("tlora_tp_create", C.byref(desc), comm, C.byref(h))
        self._h = h
        self.layers = {}
        for p, (name, d, k) in enumerate(wl.projections):
            lh = C.c_void_p()
            call("tlora_tp_layer", self._h, p, C.byref(lh))
            dd, kk = (d // P, k) if name in ROW else (d, k // P)
            self.layers[name] = _LayerView(lh, dd, kk, wl.ranks, device)
        seed = wl.seed if seed is None else seed
        self.full_weights = {}
        for pi, (name, d, k) in enumerate(wl.projections):  # as TPLayerSetStep.__init__
            g = torch.Generator(device=self.dev).manual_seed(seed * 1000 + pi)
            W = (torch.randn(d, k, generator=g, device=self.dev) * d ** -0.5).bfloat16()
            As = [(torch.randn(d, j.rank, generator=g, device=self.dev) * d ** -0.5).bfloat16()
                  for j in wl.jobs]
            Bs = [(torch.randn(j.rank, k, generator=g, device=self.dev) * j.rank ** -0.5).bfloat16()
                  for j in wl.jobs]
            lay = self.layers[name]
            if name in COLUMN:
                lay.set_base(shard_columns(W, rank, P))
                for s in range(len(wl.jobs)):
                    lay.set_adapter(s, As[s], shard_columns(Bs[s], rank, P))
            else:
                lay.set_base(shard_rows(W, rank, P))
                for s in range(len(wl.jobs)):
                    lay.set_adapter(s, shard_rows(As[s], rank, P), Bs[s])
            self.full_weights[name] = (W, As, Bs)
        buf = self._buf
        self.X_shard = {g: buf(BUF_X_SHARD, i) for i, g in enumerate(self.groups)}
        self.dX_shard = {g: buf(BUF_DX_SHARD, i) for i, g in enumerate(self.groups)}
        self.Y, self.dY, self.X_loc, self.dY_shard, self.Y_shard, self.dX_loc = {}, {}, {}, {}, {}, {}
        for p, name in enumerate(names):
            if name in COLUMN:
                self.Y[name], self.dY[name] = buf(BUF_Y, p), buf(BUF_DY, p)
            else:
                self.X_loc[name], self.dY_shard[name] = buf(BUF_X_LOC, p), buf(BUF_DY_SHARD, p)
                self.Y_shard[name], self.dX_loc[name] = buf(BUF_Y_SHARD, p), buf(BUF_DX_LOC, p)
        # the Python driver's input draws, in its order
        gen = torch.Generator(device=self.dev).manual_seed(seed * 7919 + rank)
        rnd = lambda *shape: torch.randn(*shape, generator=gen, device=self.dev).bfloat16()  # noqa: E731
        T = wl.tokens
        for g in self.groups:
            self.X_shard[g].copy_(rnd(*self.X_shard[g].shape))
        for name in COLUMN:
            if name in names:
                self.dY[name].copy_(rnd(*self.dY[name].shape))
        for name in ROW:
            if name in names:
                self.X_loc[name].copy_(rnd(*self.X_loc[name].shape))
                self.dY_shard[name].copy_(rnd(*self.dY_shard[name].shape))
        self.T = T
        torch.cuda.synchronize(self.dev)

    def _buf(self, kind, index):
        p, r, c = C.c_void_p(), C.c_int64(), C.c_int64()
        call("tlora_tp_buffer", self._h, kind, index, C.byref(p), C.byref(r), C.byref(c))
        return _torch_view(p.value, r.value, c.value, torch.bfloat16, self.dev)

    def enable_optimizer(self, base_lr: float = 1e-4, weight_decay: float = 0.01):
        lrs = [base_lr * (1.0 + 0.25 * (s % 4)) for s in range(len(self.wl.jobs))]
        for lay in self.layers.values():
            lay.set_optimizer(lrs, weight_decay)

    def layout(self, n: int):
        S = len(self.wl.jobs)
        m = max(1, min(n, sum(j.batch for j in self.wl.jobs)))
        t0 = np.zeros(m + 1, np.int64)
        ns = np.zeros(m * S, np.int32)
        out = C.c_int32()
        call("tlora_tp_layout", self._h, int(n), C.byref(out), t0.ctypes.data, ns.ctypes.data)
        return out.value, t0, ns.reshape(m, S)

    def run(self, stream=None, trace: bool = False) -> StepStats:
        st = capi.StepStatsC()
        call("tlora_tp_run", self._h, capi.RUN_TRACE if trace else 0, _stream_ptr(stream),
             C.byref(st))
        return StepStats(st.nano_used, st.next_nano, st.ms, False, st.launches, st.tokens)

    def trace(self):
        """(t_comp_ms, t_comm_ms) per nano-batch of the last run(trace=True)."""
        n = C.c_int32()
        call("tlora_tp_trace", self._h, None, None, 0, C.byref(n))
        a = (C.c_double * max(1, n.value))()
        b = (C.c_double * max(1, n.value))()
        call("tlora_tp_trace", self._h, a, b, n.value, C.byref(n))
        return list(a[: n.value]), list(b[: n.value])

    def close(self):
        if getattr(self, "_h", None):
            capi.lib().tlora_tp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
