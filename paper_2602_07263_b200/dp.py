"""Data-parallel adapter-gradient all-reduce by copy-engine push (DP replicas).

NCCL's all-reduce kernels need SMs, and during the backward every SM is held by a
persistent fused GEMM, so the overlapped all-reduce and the GEMMs slow each other down.
Here the exchange is a reduce-scatter then an all-gather, both by cudaMemcpyAsync pushes
into peers' symmetric buffers (copy engines over NVLink/NVSwitch, no SM), each phase
closed by flags in every peer's flag array (cuStreamWriteValue32, fenced after the
copies; cuStreamWaitValue32 on the receiver). The owner of a chunk sums its P slots in slot
order and distributes the result, so the replicas' gradients stay bitwise identical.

Receive buffers are double-buffered by step parity: a rank pushes step s+1's gradients of
a projection while a slower peer may still be summing step s's; it can only come back to
the same parity after consuming that peer's step s+1 flags, which the peer raised after
its step s sums (same comm stream). Memory: 2 x 2 x (gradient bytes) per rank.
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from .capi import call


class PushAllReduce:
    def __init__(self, world: int, rank: int, device, group=None):
        import torch.distributed._symmetric_memory as symm_mem
        self.symm = symm_mem
        self.P, self.rank, self.dev = world, rank, torch.device(device)
        self.group = group if group is not None else dist.group.WORLD
        self.flags = symm_mem.empty(world, dtype=torch.int32, device=self.dev)
        self.flags.zero_()
        self.flag_hdl = symm_mem.rendezvous(self.flags, self.group)
        self.bufs = {}   # key -> (n, chunk, recv [2, P, chunk], handle, res [2, P*chunk], handle)
        self.epoch = 0
        self.parity = 0
        torch.cuda.synchronize(self.dev)
        dist.barrier(group=self.group)

    def register(self, key, n: int):
        c = (n + self.P - 1) // self.P
        c = (c + 3) // 4 * 4  # 16-byte aligned chunks
        recv = self.symm.empty(2, self.P, c, dtype=torch.float32, device=self.dev)
        res = self.symm.empty(2, self.P * c, dtype=torch.float32, device=self.dev)
        self.bufs[key] = (n, c, recv, self.symm.rendezvous(recv, self.group), res,
                          self.symm.rendezvous(res, self.group))

    def next_step(self):
        self.parity ^= 1

    @staticmethod
    def _pieces(tensors, lo, hi):
        """(tensor, element offset, count) pieces of the virtual concatenation [lo, hi)."""
        out, base = [], 0
        for t in tensors:
            n = t.numel()
            a, b = max(lo, base), min(hi, base + n)
            if a < b:
                out.append((t, a - base, b - a))
            base += n
        return out

    def _flag_and_wait(self, sp):
        P, r = self.P, self.rank
        self.epoch += 1
        for q in range(P):
            if q != r:
                call("tlora_stream_write_u32", sp,
                     C.c_void_p(int(self.flag_hdl.buffer_ptrs[q]) + 4 * r), self.epoch)
        fb = self.flags.data_ptr()
        for q in range(P):
            if q != r:
                call("tlora_stream_wait_u32", sp, C.c_void_p(fb + 4 * q), self.epoch)

    def allreduce(self, key, tensors, stream):
        """Sum `tensors` (fp32, contiguous; concatenated size = the registered n) over the
        replicas, in place, enqueued on `stream`. Two copy-engine phases with the ring's
        traffic: (1) chunk q of every rank's gradients -> rank q's receive slot, rank q sums
        its P slots in slot order; (2) every reduced chunk -> every rank's result buffer,
        copied back into `tensors`. Each chunk is summed once, by its owner, so all
        replicas end with identical bits."""
        n, c, recv, rh, res, sh = self.bufs[key]
        P, r, par = self.P, self.rank, self.parity
        sp = C.c_void_p(stream.cuda_stream)
        # phase 1: my chunk q -> recv[par][slot r] on rank q
        for j in range(P):  # ring order from the next rank; self last
            q = (r + 1 + j) % P
            lo, hi = q * c, min(n, (q + 1) * c)
            dst = int(rh.buffer_ptrs[q]) + ((par * P + r) * c) * 4
            off = 0
            for t, a, cnt in self._pieces(tensors, lo, hi):
                call("tlora_copy_async", C.c_void_p(dst + off * 4),
                     C.c_void_p(t.data_ptr() + a * 4), C.c_size_t(cnt * 4), sp)
                off += cnt
        self._flag_and_wait(sp)
        lo, hi = r * c, min(n, (r + 1) * c)
        with torch.cuda.stream(stream):
            if hi > lo:
                torch.sum(recv[par, :, :hi - lo], dim=0, out=res[par, lo:hi])
        # phase 2: my reduced chunk -> res[par][lo:hi] on every peer
        for j in range(P - 1):
            q = (r + 1 + j) % P
            if hi > lo:
                call("tlora_copy_async", C.c_void_p(int(sh.buffer_ptrs[q]) + (par * P * c + lo) * 4),
                     C.c_void_p(res[par, lo:hi].data_ptr()), C.c_size_t((hi - lo) * 4), sp)
        self._flag_and_wait(sp)
        with torch.cuda.stream(stream):
            base = 0
            for t in tensors:
                k = t.numel()
                t.view(-1).copy_(res[par, base:base + k])
                base += k
