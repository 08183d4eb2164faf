"""C-ABI communicator check (run under torchrun with >= 2 GPUs, one rank per GPU).

Rank 0 makes the NCCL unique id through tlora_comm_get_unique_id, torch.distributed (gloo)
broadcasts it, every rank creates a tlora communicator (world = tp * dp with tp = 2 when
the world is even, so TP and DP groups are both exercised) and checks, against
torch.distributed on the same data:
  * tlora_layer_allreduce_grads over the DP group (sum and mean): bitwise equal to the
    fp32 sum / mean of every DP peer's gradients gathered with torch;
  * tlora_comm_all_gather / reduce_scatter over the TP group (bf16) and all_reduce over
    the world: equal to the torch-gathered reference (sums of 2 bf16 values are exact in
    fp32 and rounded once, as NCCL does).

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tests/comm_check.py
"""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_07263_b200 import capi  # noqa: E402
from paper_2602_07263_b200.layer import FusedLoRALayer  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    tp = 2 if world % 2 == 0 and world > 2 else 1
    dp = world // tp
    uid = torch.zeros(capi.UNIQUE_ID_BYTES, dtype=torch.uint8)
    if rank == 0:
        buf = (C.c_uint8 * capi.UNIQUE_ID_BYTES)()
        capi.call("tlora_comm_get_unique_id", buf)
        uid = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
    dist.broadcast(uid, 0)
    idb = (C.c_uint8 * capi.UNIQUE_ID_BYTES)(*uid.tolist())
    h = C.c_void_p()
    capi.call("tlora_comm_create", local, idb, world, rank, tp, C.byref(h))
    info = [C.c_int32() for _ in range(4)]
    capi.call("tlora_comm_info", h, *[C.byref(x) for x in info])
    assert [x.value for x in info] == [world, rank, tp, dp], [x.value for x in info]
    s = torch.cuda.current_stream().cuda_stream
    bad = []

    # ---- DP gradient all-reduce of a real layer after one backward
    d, k, ranks = 256, 384, [8, 24, 64]
    dev = torch.device("cuda", local)
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    lay = FusedLoRALayer(d, k, ranks, device=local)
    lay.set_base((torch.randn(d, k, generator=g, device=dev) * 0.05).bfloat16())
    for sl, r in enumerate(ranks):
        lay.set_adapter(sl, (torch.randn(d, r, generator=g, device=dev) * 0.05).bfloat16(),
                        (torch.randn(r, k, generator=g, device=dev) * 0.05).bfloat16())
    slots = np.repeat(np.arange(3), [100, 37, 200]).astype(np.int32)
    plan = lay.plan(slots)
    X = torch.randn(len(slots), d, generator=g, device=dev).bfloat16()
    dY = torch.randn(len(slots), k, generator=g, device=dev).bfloat16()
    Y, H = lay.forward(plan, X)
    lay.backward(plan, dY, X, H)
    torch.cuda.synchronize()
    mine = [t.clone().cpu() for t in lay.packed_grads()]
    allg = [[torch.empty_like(t) for _ in range(world)] for t in mine]
    for t, lst in zip(mine, allg):
        dist.all_gather(lst, t)
    dp_peers = [p for p in range(world) if p % tp == rank % tp]
    for average in (0, 1):
        lay_grads = lay.packed_grads()
        for t, m in zip(lay_grads, mine):  # restore this rank's own grads
            t.copy_(m.to(dev))
        capi.call("tlora_layer_allreduce_grads", lay._h, h, capi.GROUP_DP, average, s)
        torch.cuda.synchronize()
        for i, t in enumerate(lay.packed_grads()):
            ref = allg[i][dp_peers[0]].clone()
            for p in dp_peers[1:]:
                ref += allg[i][p]
            if average:
                ref /= len(dp_peers)
            got = t.cpu()
            if not (torch.equal(got, ref) if len(dp_peers) <= 2 and not average
                    else torch.allclose(got, ref, rtol=1e-6, atol=1e-7)):
                bad.append(f"grads[{i}] average={average} max|d|={(got - ref).abs().max().item():.3e}")

    # ---- TP all-gather / reduce-scatter (bf16) and world all-reduce
    n = 4096
    x = (torch.randn(n, generator=g, device=dev) * (rank + 1)).bfloat16()
    xs = [torch.empty_like(x.cpu()) for _ in range(world)]
    dist.all_gather(xs, x.cpu())
    tp_peers = [p for p in range(world) if p // tp == rank // tp]
    ag = torch.empty(n * tp, dtype=torch.bfloat16, device=dev)
    capi.call("tlora_comm_all_gather", h, capi.GROUP_TP, x.data_ptr(), ag.data_ptr(), n,
              capi.BF16, s)
    rsd = torch.empty(n // tp, dtype=torch.bfloat16, device=dev)
    capi.call("tlora_comm_reduce_scatter", h, capi.GROUP_TP, x.data_ptr(), rsd.data_ptr(), n // tp,
              capi.BF16, s)
    ar = torch.empty(n, dtype=torch.bfloat16, device=dev)
    capi.call("tlora_comm_all_reduce", h, capi.GROUP_WORLD, x.data_ptr(), ar.data_ptr(), n,
              capi.BF16, 0, s)
    torch.cuda.synchronize()
    if not torch.equal(ag.cpu(), torch.cat([xs[p] for p in tp_peers])):
        bad.append("all_gather")
    ti = tp_peers.index(rank)
    rs_ref = sum(xs[p].float() for p in tp_peers).bfloat16()[ti * (n // tp):(ti + 1) * (n // tp)]
    if tp == 2 and not torch.equal(rsd.cpu(), rs_ref):
        bad.append("reduce_scatter")
    if tp == 1 and not torch.equal(rsd.cpu(), x.cpu()):
        bad.append("reduce_scatter (tp=1 identity)")
    # NCCL reduces bf16 in bf16: every partial sum of the ring/tree is rounded (half an ulp,
    # 2^-9 relative), so after world-1 additions and the final store the error is bounded by
    # world * 2^-9 * sum_p |x_p| (x2 margin below). Exact for world = 2 (one rounding).
    ar_ref = sum(xs[p].float() for p in range(world))
    ar_bound = world * 2.0 ** -8 * sum(xs[p].float().abs() for p in range(world)) + 1e-6
    ar_err = (ar.cpu().float() - ar_ref).abs()
    if not bool((ar_err <= ar_bound).all()):
        bad.append(f"all_reduce max|d|={ar_err.max().item():.3e} "
                   f"worst ratio={(ar_err / ar_bound).max().item():.2f}")
    capi.call("tlora_comm_destroy", h)
    lay.close()
    ok = torch.tensor([0 if bad else 1])
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if bad:
        print(f"rank{rank} FAIL: {bad}", flush=True)
    if rank == 0:
        print("COMM_CHECK", "PASS" if ok.item() == 1 else "FAIL", f"world={world} tp={tp} dp={dp}",
              flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok.item() == 1 else 1)


if __name__ == "__main__":
    main()
