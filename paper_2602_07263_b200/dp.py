"""Data-parallel adapter-gradient all-reduce by copy-engine push (DP replicas).

NCCL's all-reduce kernels need SMs, and during the backward every SM is held by a
persistent fused GEMM, so the overlapped all-reduce and the GEMMs slow each other down.
Here each rank pushes its packed fp32 gradients into slot `rank` of every peer's receive
buffer with cudaMemcpyAsync (copy engines over NVLink/NVSwitch, no SM), raises its flag in
every peer's flag array (cuStreamWriteValue32, fenced after the copies), waits for all
peers' flags (cuStreamWaitValue32), and sums the P slots in slot order. Every rank sums the
same P slots in the same order, so the replicas' gradients stay bitwise identical.

Receive buffers are double-buffered by step parity: a rank pushes step s+1's gradients of
a projection while a slower peer may still be summing step s's; it can only come back to
the same parity after consuming that peer's step s+1 flags, which the peer raised after
its step s sums (same comm stream). Memory: 2 x P x (gradient bytes) per rank.
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
        self.bufs = {}   # key -> (recv [2, P, n] fp32, handle)
        self.epoch = 0
        self.parity = 0
        torch.cuda.synchronize(self.dev)
        dist.barrier(group=self.group)

    def register(self, key, n: int):
        buf = self.symm.empty(2, self.P, n, dtype=torch.float32, device=self.dev)
        self.bufs[key] = (buf, self.symm.rendezvous(buf, self.group))

    def next_step(self):
        self.parity ^= 1

    def allreduce(self, key, tensors, stream):
        """Sum `tensors` (fp32, contiguous; concatenated size = the registered n) over the
        replicas, in place, enqueued on `stream`."""
        buf, hdl = self.bufs[key]
        P, r = self.P, self.rank
        n = buf.shape[2]
        sp = C.c_void_p(stream.cuda_stream)
        slot_bytes, plane_bytes = n * 4, P * n * 4
        base_off = self.parity * plane_bytes + r * slot_bytes
        for j in range(P):  # ring order from the next rank; self last
            q = (r + 1 + j) % P
            off = 0
            for t in tensors:
                nb = t.numel() * 4
                call("tlora_copy_async", C.c_void_p(int(hdl.buffer_ptrs[q]) + base_off + off),
                     C.c_void_p(t.data_ptr()), C.c_size_t(nb), sp)
                off += nb
        self.epoch += 1
        for q in range(P):
            if q != r:
                call("tlora_stream_write_u32", sp,
                     C.c_void_p(int(self.flag_hdl.buffer_ptrs[q]) + 4 * r), self.epoch)
        fb = self.flags.data_ptr()
        for q in range(P):
            if q != r:
                call("tlora_stream_wait_u32", sp, C.c_void_p(fb + 4 * q), self.epoch)
        with torch.cuda.stream(stream):
            total = buf[self.parity].sum(dim=0)  # slot order 0..P-1 on every rank
            off = 0
            for t in tensors:
                k = t.numel()
                t.view(-1).copy_(total[off:off + k])
                off += k
