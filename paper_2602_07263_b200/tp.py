"""Tensor-parallel fused multi-LoRA layer set with rank-aware nano-batches.

One process per GPU; the P ranks of the group split W (Megatron style, sequence-parallel
activations between projection groups):

  column-parallel  q, k, v, gate, up   W[:, k/P], B_j[:, k/P] local, A_j replicated
      fwd: shrink on this rank's token shard -> all-gather [X | H] -> fused GEMM (local N)
      bwd: dH_p = dY_p·B_pᵀ and dX_p = dY_p·W_pᵀ + dH_p·Aᵀ are partial sums over ranks;
           reduce-scatter [dX | dH] (dX of projections sharing an input summed in place
           first), dA_j from the token shard (all-reduced over TP once per step),
           dB_j local from the gathered H.
  row-parallel     o, down             W[d/P, :], A_j[d/P, :] local, B_j replicated
      fwd: partial H_p = X_p·A_p and Y_p = X_p·W_p + H_p·B; reduce-scatter Y
      bwd: all-gather dY; dH = dY·Bᵀ exact; dX local; dA_j local; dB_j partial
           (all-reduced over TP once per step).

The combined batch (Σ_j B_j samples) is cut into N nano-batches with the reference's
balanced `partition` counts (nano_pipeline.hpp:51-60) and the rank-aware map of the step
executor (tlora_nano_assign: LoRA work balanced across nano-batches); every nano-batch is
job-contiguous (the fast case of the tile packer). A compute stream runs the tlora
launches and a comm stream runs the NCCL collectives: the all-gather of nano n+1 and the
reduce-scatter of nano n-1 overlap the GEMMs of nano n. N is adapted online by the
reference's AIMD rule (nano_pipeline.hpp:99-112) from CUDA-event step times — the real
version of the simulator loop sim_engine.hpp:306-315.

Inputs of the four projection groups are independent synthetic activations (attention,
norms and activations are outside the path); the collective pattern is the real one.
"""
from __future__ import annotations

import ctypes as _C
import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .capi import call as _call
from .layer import AimdState, FusedLoRALayer, aimd_step, partition, reduce_slots
from .workload import INPUT_GROUP, Workload

COLUMN = ("q", "k", "v", "gate", "up")
ROW = ("o", "down")


# ------------------------------------------------------------------ pure host-side plan
@dataclass
class NanoBatch:
    index: int
    t0: int          # first global token of this nano-batch (nano order)
    tokens: int      # T_n
    slots: np.ndarray  # owning slot per token, job-contiguous

    def shard(self, rank: int, world: int):
        """(first row within the nano, rows) of this rank's sequence-parallel shard."""
        assert self.tokens % world == 0
        n = self.tokens // world
        return rank * n, n


def nano_batches(wl: Workload, n: int) -> list[NanoBatch]:
    """partition(Σ_j B_j, n) samples into nano-batches with the executor's rank-aware map
    (tlora_nano_assign: partition's counts, per-sample work balanced across nano-batches,
    each (nano, job) a contiguous range of the job's samples); inside a nano-batch the jobs
    stay contiguous in slot order, the fast case of the tile packer."""
    from .step import nano_assign, sample_weights
    batch = [j.batch for j in wl.jobs]
    k, per, _, ns = nano_assign(batch, sample_weights(wl), n)
    out, t0 = [], 0
    for idx in range(k):
        slots = np.concatenate([np.full(int(ns[idx, s]) * j.seq_len, s, np.int32)
                                for s, j in enumerate(wl.jobs)])
        out.append(NanoBatch(idx, t0, int(slots.shape[0]), slots))
        t0 += int(slots.shape[0])
    return out


def shard_columns(full: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    k = full.shape[1]
    assert k % world == 0
    w = k // world
    return full[:, rank * w:(rank + 1) * w].contiguous()


def shard_rows(full: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    d = full.shape[0]
    assert d % world == 0
    w = d // world
    return full[rank * w:(rank + 1) * w].contiguous()


# ------------------------------------------------------------------ the driver
class TPLayerSetStep:
    def __init__(self, wl: Workload, rank: int, world: int, device: int, group=None,
                 nano: int = 4, seed: int | None = None, fused_rs=False):
        self.wl, self.rank, self.world, self.group = wl, rank, world, group
        self.dev = torch.device("cuda", device)
        self.T = wl.tokens
        self.n = nano
        self.compute = torch.cuda.current_stream(self.dev)
        self.comm = torch.cuda.Stream(self.dev)
        # collectives and the side-stream gradient launches take SMs from the persistent
        # fused GEMMs: dynamic tile scheduling keeps them balanced (C4 TP4: 33.6 -> 32.0 ms)
        if "TLORA_DYN_SCHED" not in os.environ:
            _call("tlora_set_tile_scheduler", device, 1)
        # adapter-gradient launches (HBM-bound) run on their own stream, overlapping the
        # fused GEMMs of the compute stream (as runner.LayerSetStep.enable_side_grads)
        self.gside = (torch.cuda.Stream(self.dev) if os.environ.get("TLORA_TP_SIDE_GRADS", "1") != "0"
                      else self.compute)
        seed = wl.seed if seed is None else seed
        self.layers, self.R = {}, {}
        self.full_weights = {}
        P, T = world, self.T
        bf = torch.bfloat16
        for pi, (name, d, k) in enumerate(wl.projections):
            # identical full weights on every rank (same seed), then this rank's slice
            g = torch.Generator(device=self.dev).manual_seed(seed * 1000 + pi)
            W = (torch.randn(d, k, generator=g, device=self.dev) * d ** -0.5).bfloat16()
            As = [(torch.randn(d, j.rank, generator=g, device=self.dev) * d ** -0.5).bfloat16()
                  for j in wl.jobs]
            Bs = [(torch.randn(j.rank, k, generator=g, device=self.dev) * j.rank ** -0.5).bfloat16()
                  for j in wl.jobs]
            if name in COLUMN:
                lay = FusedLoRALayer(d, k // P, wl.ranks, device=device)
                lay.set_base(shard_columns(W, rank, P))
                for s in range(len(wl.jobs)):
                    lay.set_adapter(s, As[s], shard_columns(Bs[s], rank, P))
            else:
                lay = FusedLoRALayer(d // P, k, wl.ranks, device=device)
                lay.set_base(shard_rows(W, rank, P))
                for s in range(len(wl.jobs)):
                    lay.set_adapter(s, shard_rows(As[s], rank, P), Bs[s])
            self.layers[name] = lay
            self.R[name] = lay.R
            self.full_weights[name] = (W, As, Bs)
        # step-sized buffers; nano-batch n is a row range of each (no realloc when N moves)
        gen = torch.Generator(device=self.dev).manual_seed(seed * 7919 + rank)
        rnd = lambda *shape: torch.randn(*shape, generator=gen, device=self.dev).to(bf)  # noqa: E731
        dims = {name: (d, k) for name, d, k in wl.projections}
        self.groups = sorted({INPUT_GROUP[p] for p in COLUMN if p in dims})
        gdim = {INPUT_GROUP[p]: dims[p][0] for p in COLUMN if p in dims}
        self.X_shard = {g: rnd(T // P, gdim[g]) for g in self.groups}
        self.X_full = {g: torch.empty(T, gdim[g], dtype=bf, device=self.dev) for g in self.groups}
        self.dX_part = {g: torch.empty(T, gdim[g], dtype=bf, device=self.dev) for g in self.groups}
        self.dX_shard = {g: torch.empty(T // P, gdim[g], dtype=bf, device=self.dev)
                         for g in self.groups}
        self.H_shard, self.H_full, self.Y, self.dY, self.dH_part, self.dH_shard = {}, {}, {}, {}, {}, {}
        self.X_loc, self.H_row, self.Y_part, self.Y_shard, self.dY_shard, self.dY_full = ({}, {}, {},
                                                                                         {}, {}, {})
        self.dH_row, self.dX_loc = {}, {}
        for name in COLUMN:
            if name not in dims:
                continue
            d, k = dims[name]
            R = self.R[name]
            self.H_shard[name] = torch.empty(T // P, R, dtype=bf, device=self.dev)
            self.H_full[name] = torch.empty(T, R, dtype=bf, device=self.dev)
            self.Y[name] = torch.empty(T, k // P, dtype=bf, device=self.dev)
            self.dY[name] = rnd(T, k // P)
            self.dH_part[name] = torch.empty(T, R, dtype=bf, device=self.dev)
            self.dH_shard[name] = torch.empty(T // P, R, dtype=bf, device=self.dev)
        for name in ROW:
            if name not in dims:
                continue
            d, k = dims[name]
            R = self.R[name]
            self.X_loc[name] = rnd(T, d // P)
            self.H_row[name] = torch.empty(T, R, dtype=bf, device=self.dev)
            self.Y_part[name] = torch.empty(T, k, dtype=bf, device=self.dev)
            self.Y_shard[name] = torch.empty(T // P, k, dtype=bf, device=self.dev)
            self.dY_shard[name] = rnd(T // P, k)
            self.dY_full[name] = torch.empty(T, k, dtype=bf, device=self.dev)
            self.dH_row[name] = torch.empty(T, R, dtype=bf, device=self.dev)
            self.dX_loc[name] = torch.empty(T, d // P, dtype=bf, device=self.dev)
        self._plans = {}
        self.aimd = AimdState(n=nano)
        # fused GEMM + reduce-scatter for the row-parallel projections: every rank's receive
        # buffer [world][T/P][k] in symmetric (peer-mapped) memory
        # fused_rs: False, True (all row-parallel projections) or a collection of names
        if fused_rs is True:
            fused_rs = ROW
        self.fused_set = set(fused_rs or ())
        self.fused_rs = bool(self.fused_set)
        self.recv, self.recv_hdl = {}, {}
        if self.fused_rs:
            import torch.distributed._symmetric_memory as symm_mem
            grp = group if group is not None else dist.group.WORLD
            for name in ROW:
                if name not in dims or name not in self.fused_set:
                    continue
                k = dims[name][1]
                buf = symm_mem.empty(P, T // P, k, dtype=bf, device=self.dev)
                self.recv[name] = buf
                self.recv_hdl[name] = symm_mem.rendezvous(buf, grp)
        # Copy-engine all-gather (TLORA_TP_CE_AG, default on at P > 1). NCCL's all-gather
        # kernels need SMs that the persistent fused GEMMs hold for their whole launch (at
        # TP4 a nano-batch's boundary traffic took ~6 ms, as long as its compute). Here the
        # gathered buffers live in symmetric (peer-mapped) memory; each rank pushes its
        # shard rows into every peer's buffer with cudaMemcpyAsync on the comm stream (copy
        # engines over NVLink, no SM), then raises its flag in each peer's flag array
        # (cuStreamWriteValue32, fenced after the copies). The consumer's compute stream
        # waits for every peer's flag to reach the gather's epoch (cuStreamWaitValue32).
        # Epochs advance identically on all ranks (same gather sequence). Buffer reuse is
        # ordered by the step structure: a rank pushes into a buffer only after it consumed
        # a later flag of that peer, raised after the peer's last read of the buffer.
        # (TLORA_TP_CE_SELF=1 keeps it at P = 1: pushes to this rank's own buffers, the
        # single-GPU test coverage of the copy-engine data path)
        self.ce_ag = ((P > 1 or os.environ.get("TLORA_TP_CE_SELF") == "1")
                      and os.environ.get("TLORA_TP_CE_AG", "1") != "0")
        self.ag_hdl = {}
        if self.ce_ag:
            import torch.distributed._symmetric_memory as symm_mem
            grp = group if group is not None else dist.group.WORLD

            def symm(key, like):
                buf = symm_mem.empty(*like.shape, dtype=like.dtype, device=self.dev)
                self.ag_hdl[key] = symm_mem.rendezvous(buf, grp)
                return buf

            for g in self.groups:
                self.X_full[g] = symm(("X", g), self.X_full[g])
            for name in list(self.H_full):
                self.H_full[name] = symm(("H", name), self.H_full[name])
            for name in list(self.dY_full):
                self.dY_full[name] = symm(("dY", name), self.dY_full[name])
            # reduce-scatter by push: receive slots [P][T/P][width] (slot = source rank);
            # every rank copies its partial rows of owner q's shard into q's slot, then the
            # owner sums the P slots in fixed order (reduce_slots, deterministic)
            self.rs_recv = {}
            for g in self.groups:
                w = self.dX_shard[g].shape[1]
                self.rs_recv[("rsX", g)] = symm(("rsX", g), torch.empty(P, T // P, w, dtype=bf))
            for name in list(self.dH_shard):
                w = self.dH_shard[name].shape[1]
                self.rs_recv[("rsH", name)] = symm(("rsH", name), torch.empty(P, T // P, w, dtype=bf))
            self.flags = symm_mem.empty(P, dtype=torch.int32, device=self.dev)
            self.flags.zero_()
            self.flag_hdl = symm_mem.rendezvous(self.flags, grp)
            self._epoch = 0
            torch.cuda.synchronize(self.dev)
            dist.barrier(group=grp)  # every rank's flags are zero before any push
        torch.cuda.synchronize(self.dev)

    def _ag_ce(self, stream, items, b) -> int:
        """Push this rank's rows of nano-batch b into every rank's gathered buffers (the
        all_gather_into_tensor layout: rank r's shard at rows b.t0 + r * b.tokens / P),
        then raise this rank's flag on every peer. Returns the epoch to wait for."""
        P, r = self.world, self.rank
        nr = b.tokens // P
        sp = _C.c_void_p(stream.cuda_stream)
        for key, full, shard in items:
            row_bytes = full.shape[1] * full.element_size()
            off, nbytes = (b.t0 + r * nr) * row_bytes, nr * row_bytes
            ptrs = self.ag_hdl[key].buffer_ptrs
            for j in range(P):  # peers first in ring order from the next rank, self last
                q = (r + 1 + j) % P
                _call("tlora_copy_async", _C.c_void_p(int(ptrs[q]) + off),
                      _C.c_void_p(shard.data_ptr()), _C.c_size_t(nbytes), sp)
        self._epoch += 1
        for q in range(P):
            if q != r:
                _call("tlora_stream_write_u32", sp,
                      _C.c_void_p(int(self.flag_hdl.buffer_ptrs[q]) + 4 * r), self._epoch)
        return self._epoch

    def _rs_ce(self, stream, items, b):
        """Reduce-scatter of nano-batch b by copy-engine push: for each (key, partial rows
        [b.tokens x w], output shard rows [b.tokens / P x w]) this rank copies the chunk
        owned by rank q into q's receive slot `rank`, raises its flags, waits for every
        peer's, and sums its own P slots (reduce_slots) into the output, all on `stream`."""
        P, r = self.world, self.rank
        nr, slot_rows, row0 = b.tokens // P, self.T // P, b.t0 // P
        sp = _C.c_void_p(stream.cuda_stream)
        for key, part, out in items:
            w = part.shape[1]
            row_bytes = w * part.element_size()
            ptrs = self.ag_hdl[key].buffer_ptrs
            dst_off = (r * slot_rows + row0) * row_bytes
            for j in range(P):
                q = (r + 1 + j) % P
                _call("tlora_copy_async", _C.c_void_p(int(ptrs[q]) + dst_off),
                      _C.c_void_p(part.data_ptr() + q * nr * row_bytes),
                      _C.c_size_t(nr * row_bytes), sp)
        self._epoch += 1
        for q in range(P):
            if q != r:
                _call("tlora_stream_write_u32", sp,
                      _C.c_void_p(int(self.flag_hdl.buffer_ptrs[q]) + 4 * r), self._epoch)
        self._ag_wait(stream, self._epoch)
        for key, part, out in items:
            recv = self.rs_recv[key]
            reduce_slots(recv, P, slot_rows, row0, nr, recv.shape[2], out, stream=stream)

    def _ag_wait(self, stream, epoch):
        sp = _C.c_void_p(stream.cuda_stream)
        base = self.flags.data_ptr()
        for q in range(self.world):
            if q != self.rank:
                _call("tlora_stream_wait_u32", sp, _C.c_void_p(base + 4 * q), epoch)

    # -------------------------------------------------------------- plans per N
    def plans(self, n: int):
        if n not in self._plans:
            nb = nano_batches(self.wl, n)
            per = []
            for b in nb:
                r0, rows = b.shard(self.rank, self.world)
                shard_slots = b.slots[r0:r0 + rows]
                per.append({name: (lay.plan(b.slots),
                                   lay.plan(shard_slots) if name in COLUMN else None)
                            for name, lay in self.layers.items()})
            self._plans[n] = (nb, per)
        return self._plans[n]

    # -------------------------------------------------------------- helpers
    def _rows(self, t, b: NanoBatch):
        return t[b.t0:b.t0 + b.tokens]

    def _srows(self, t, b: NanoBatch):
        return t[b.t0 // self.world:(b.t0 + b.tokens) // self.world]

    def _ag(self, out, inp):
        dist.all_gather_into_tensor(out, inp, group=self.group)

    def _rs(self, out, inp):
        dist.reduce_scatter_tensor(out, inp, group=self.group)

    # -------------------------------------------------------------- pipeline trace
    def enable_trace(self, on: bool = True):
        """Record CUDA events around every nano-batch's compute (compute stream) and
        boundary traffic (comm stream) — the measured PipelineTrace of the reference's
        monitor (nano_pipeline.hpp:28-34, 114-126)."""
        self._trace = {} if on else None

    def _mark(self, stream, kind: str, i: int, edge: int):
        tr = getattr(self, "_trace", None)
        if tr is None:
            return
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        tr.setdefault((kind, i), [None, None])[edge] = e

    def trace_reading(self, step_ms: float):
        """PipelineTrace of the last traced step (seconds): t_comp / t_comm per nano-batch
        (forward + backward intervals summed), t_iter_event = the measured step time,
        t_iter_analytic = max(sum t_comp, sum t_comm) (the overlap ideal); and the
        reference's monitor() of it."""
        torch.cuda.synchronize(self.dev)
        comp, comm = {}, {}
        for (kind, i), (e0, e1) in self._trace.items():
            if e0 is None or e1 is None:
                continue
            dst = comp if kind.startswith("comp") else comm
            dst[i] = dst.get(i, 0.0) + e0.elapsed_time(e1) / 1e3
        n = max(list(comp) + list(comm)) + 1 if comp or comm else 0
        t_comp = [comp.get(i, 0.0) for i in range(n)]
        t_comm = [comm.get(i, 0.0) for i in range(n)]
        t_event = step_ms / 1e3
        t_analytic = max(sum(t_comp), sum(t_comm))
        from .layer import monitor
        eta, stall = monitor(t_comp, t_comm, t_event, t_analytic, num_stages=1)
        return {"t_comp_s": t_comp, "t_comm_s": t_comm, "t_iter_event_s": t_event,
                "t_iter_analytic_s": t_analytic, "eta_util": eta, "delta_stall_s": stall}

    # -------------------------------------------------------------- forward
    def forward(self, n: int | None = None):
        n = self.n if n is None else n
        nb, plans = self.plans(n)
        C, M = self.compute, self.comm
        cols = [p for p in COLUMN if p in self.layers]
        rows = [p for p in ROW if p in self.layers]
        if self.fused_rs:  # every rank has consumed the previous step's receive slots
            C.wait_stream(M)
            with torch.cuda.stream(C):
                for p in rows:
                    if p in self.fused_set:
                        self.recv_hdl[p].barrier(channel=0, timeout_ms=60000)

        def shrink(i):
            b = nb[i]
            for p in cols:
                self.layers[p].shrink(plans[i][p][1], self._srows(self.X_shard[INPUT_GROUP[p]], b),
                                      self._srows(self.H_shard[p], b), stream=C)
            ev = torch.cuda.Event()
            ev.record(C)
            return ev

        def gather(i, ev):
            b = nb[i]
            M.wait_event(ev)
            self._mark(M, "comm_ag_f", i, 0)
            epoch = None
            with torch.cuda.stream(M):
                if self.ce_ag:
                    items = ([(("X", g), self.X_full[g], self._srows(self.X_shard[g], b))
                              for g in self.groups] +
                             [(("H", p), self.H_full[p], self._srows(self.H_shard[p], b))
                              for p in cols])
                    epoch = self._ag_ce(M, items, b)
                else:
                    for g in self.groups:
                        self._ag(self._rows(self.X_full[g], b), self._srows(self.X_shard[g], b))
                    for p in cols:
                        self._ag(self._rows(self.H_full[p], b), self._srows(self.H_shard[p], b))
            self._mark(M, "comm_ag_f", i, 1)
            ev2 = torch.cuda.Event()
            ev2.record(M)
            return ev2, epoch

        ev_g = gather(0, shrink(0))
        for i in range(len(nb)):
            ev_next = gather(i + 1, shrink(i + 1)) if i + 1 < len(nb) else None
            b = nb[i]
            C.wait_event(ev_g[0])
            if ev_g[1] is not None:
                self._ag_wait(C, ev_g[1])
            self._mark(C, "comp_f", i, 0)
            for p in cols:
                self.layers[p].fused_gemm(plans[i][p][0], self._rows(self.X_full[INPUT_GROUP[p]], b),
                                          self._rows(self.H_full[p], b), self._rows(self.Y[p], b),
                                          stream=C)
            for p in rows:
                lay, pl = self.layers[p], plans[i][p][0]
                lay.shrink(pl, self._rows(self.X_loc[p], b), self._rows(self.H_row[p], b), stream=C)
                if p in self.fused_set:
                    # GEMM tiles go straight into the owners' receive slots over NVLink
                    hdl = self.recv_hdl[p]
                    lay.fused_gemm_rs(pl, self._rows(self.X_loc[p], b), self._rows(self.H_row[p], b),
                                      hdl.buffer_ptrs, self.rank, self.T // self.world,
                                      b.t0 // self.world, stream=C)
                else:
                    lay.fused_gemm(pl, self._rows(self.X_loc[p], b), self._rows(self.H_row[p], b),
                                   self._rows(self.Y_part[p], b), stream=C)
            self._mark(C, "comp_f", i, 1)
            ev_y = torch.cuda.Event()
            ev_y.record(C)
            M.wait_event(ev_y)
            self._mark(M, "comm_rs_f", i, 0)
            with torch.cuda.stream(M):  # off the compute stream: overlaps nano n+1's GEMMs
                for p in rows:
                    if p in self.fused_set:  # data already moved by the GEMM: barrier + sum
                        self.recv_hdl[p].barrier(channel=0, timeout_ms=60000)
                        reduce_slots(self.recv[p], self.world, self.T // self.world,
                                     b.t0 // self.world, b.tokens // self.world,
                                     self.recv[p].shape[2], self._srows(self.Y_shard[p], b),
                                     stream=M)
                    else:
                        self._rs(self._srows(self.Y_shard[p], b), self._rows(self.Y_part[p], b))
            self._mark(M, "comm_rs_f", i, 1)
            ev_g = ev_next
        C.wait_stream(M)

    # -------------------------------------------------------------- backward
    def backward(self, n: int | None = None):
        n = self.n if n is None else n
        nb, plans = self.plans(n)
        C, M, G = self.compute, self.comm, self.gside
        cols = [p for p in COLUMN if p in self.layers]
        rows = [p for p in ROW if p in self.layers]
        start = torch.cuda.Event()
        start.record(C)
        G.wait_event(start)

        def on_g(ev_src):  # the gradient stream waits for an event of another stream
            e = torch.cuda.Event()
            e.record(ev_src)
            G.wait_event(e)

        def gather_dy(i):
            b = nb[i]
            M.wait_event(start)
            self._mark(M, "comm_ag_b", i, 0)
            epoch = None
            with torch.cuda.stream(M):
                if self.ce_ag:
                    epoch = self._ag_ce(M, [(("dY", p), self.dY_full[p],
                                             self._srows(self.dY_shard[p], b)) for p in rows], b)
                else:
                    for p in rows:
                        self._ag(self._rows(self.dY_full[p], b), self._srows(self.dY_shard[p], b))
            self._mark(M, "comm_ag_b", i, 1)
            ev = torch.cuda.Event()
            ev.record(M)
            return ev, epoch

        def grad_a_cols(i, ev):
            b = nb[i]
            G.wait_event(ev)
            for p in cols:
                self.layers[p].grad_a(plans[i][p][1], self._srows(self.X_shard[INPUT_GROUP[p]], b),
                                      self._srows(self.dH_shard[p], b), beta=1.0 if i else 0.0,
                                      stream=G)

        ev_dy = gather_dy(0)
        pending = None
        for i in range(len(nb)):
            ev_dy_next = gather_dy(i + 1) if i + 1 < len(nb) else None
            b = nb[i]
            beta = 1.0 if i else 0.0
            C.wait_event(ev_dy[0])
            if ev_dy[1] is not None:
                self._ag_wait(C, ev_dy[1])
            self._mark(C, "comp_b", i, 0)
            # Chained schedule (as runner.LayerSetStep): each dX launch also computes the
            # NEXT projection's dH as extra tiles (tlora_backward_dx_dh), so only the first
            # dH of the nano-batch has a launch of its own. Order: row-parallel projections,
            # then the column-parallel ones in reverse.
            seq = [("row", p) for p in rows] + [("col", p) for p in reversed(cols)]

            def dy_dh(kind, p):
                if kind == "row":
                    return self._rows(self.dY_full[p], b), self._rows(self.dH_row[p], b)
                return self._rows(self.dY[p], b), self._rows(self.dH_part[p], b)

            k0, p0 = seq[0]
            dY0, dH0 = dy_dh(k0, p0)
            self.layers[p0].dh(plans[i][p0][0], dY0, dH0, stream=C)
            first = {}
            for j, (kind, p) in enumerate(seq):
                lay, pl = self.layers[p], plans[i][p][0]
                dYp, dHp = dy_dh(kind, p)
                if kind == "row":  # dH exact, dX local, dA local, dB partial
                    dXp, bx = self._rows(self.dX_loc[p], b), 0.0
                else:              # partial dH / dX (summed per input group), local dB
                    g = INPUT_GROUP[p]
                    dXp, bx = self._rows(self.dX_part[g], b), 1.0 if g in first else 0.0
                    first[g] = True
                if j + 1 < len(seq):
                    kn, pn = seq[j + 1]
                    dYn, dHn = dy_dh(kn, pn)
                    lay.dx_dh(pl, dYp, dHp, dXp, self.layers[pn], plans[i][pn][0], dYn, dHn,
                              beta=bx, zero_next=True, stream=C)
                else:
                    lay.dx(pl, dYp, dHp, dXp, beta=bx, stream=C)
                on_g(C)  # dH of p (written by the previous launch on C) and dY are ready
                if kind == "row":
                    lay.grads(pl, self._rows(self.H_row[p], b), dYp, self._rows(self.X_loc[p], b),
                              dHp, beta=beta, stream=G)
                else:
                    lay.grad_b(pl, self._rows(self.H_full[p], b), dYp, beta=beta, stream=G)
            self._mark(C, "comp_b", i, 1)
            ev_c = torch.cuda.Event()
            ev_c.record(C)
            M.wait_event(ev_c)
            self._mark(M, "comm_rs_b", i, 0)
            with torch.cuda.stream(M):
                if self.ce_ag:
                    self._rs_ce(M, [(("rsX", g), self._rows(self.dX_part[g], b),
                                     self._srows(self.dX_shard[g], b)) for g in self.groups] +
                                [(("rsH", p), self._rows(self.dH_part[p], b),
                                  self._srows(self.dH_shard[p], b)) for p in cols], b)
                else:
                    for g in self.groups:
                        self._rs(self._srows(self.dX_shard[g], b), self._rows(self.dX_part[g], b))
                    for p in cols:
                        self._rs(self._srows(self.dH_shard[p], b), self._rows(self.dH_part[p], b))
            self._mark(M, "comm_rs_b", i, 1)
            ev_r = torch.cuda.Event()
            ev_r.record(M)
            if pending is not None:
                grad_a_cols(*pending)
            pending = (i, ev_r)
            ev_dy = ev_dy_next
        grad_a_cols(*pending)
        # replicated adapter halves: sum the TP partials once per step
        C.wait_stream(G)
        ev = torch.cuda.Event()
        ev.record(C)
        M.wait_event(ev)
        with torch.cuda.stream(M):
            for p in cols:
                dist.all_reduce(self.layers[p].packed_grads()[0], group=self.group)  # dAᵀ
            for p in rows:
                dist.all_reduce(self.layers[p].packed_grads()[1], group=self.group)  # dB
        C.wait_stream(M)

    def enable_optimizer(self, base_lr: float = 1e-4, weight_decay: float = 0.01):
        lrs = [base_lr * (1.0 + 0.25 * (s % 4)) for s in range(len(self.wl.jobs))]
        for lay in self.layers.values():
            lay.set_optimizer(lrs, weight_decay)
        self.optim = True

    def step(self, n: int | None = None):
        """Training step: fwd + bwd (TP collectives) + fused AdamW of every adapter shard
        (replicated halves were all-reduced, so every rank applies identical updates)."""
        self.forward(n)
        self.backward(n)
        if getattr(self, "optim", False):
            for lay in self.layers.values():
                lay.optimizer_step(1.0, stream=self.compute)

    def adapt(self, step_seconds: float):
        """AIMD update of N from a measured step time (nano_pipeline.hpp:99-112), clamped
        to the combined batch as the simulator does (sim_engine.hpp:314)."""
        self.aimd = aimd_step(self.aimd, step_seconds)
        total = sum(j.batch for j in self.wl.jobs)
        self.aimd.n = max(1, min(self.aimd.n, total))
        self.n = self.aimd.n
        return self.n
