"""Data-parallel C++ step executor check (torchrun, >= 2 GPUs; tests/test_gpu_executor.py).

Every rank runs the executor over its own token batch with a tlora_comm (NCCL through the
C-ABI) and N = 2 nano-batches: each key's fp32 adapter gradients are all-reduced on the
executor's comm stream right after the key's last nano-batch, then AdamW applies the mean.
Checks: (1) after the step, every rank's gradient buffers equal the sum over ranks of the
gradients a communicator-less executor computes locally on the same batch (bitwise at 2
ranks; fp32 reassociation tolerance beyond); (2) all ranks hold bitwise-identical adapters
after two steps; (3) the sharded optimizer (reduce-scatter, AdamW on the owned packed-row
shard, all-gather of the bf16 operands) reproduces the all-reduce path: the next forward's
Y and the owned rows' fp32 masters are equal (bitwise at 2 ranks).
"""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from paper_2602_07263_b200.step import TrainingStep  # noqa: E402
from paper_2602_07263_b200.workload import Job, Workload  # noqa: E402

import bench  # noqa: E402  (make_comm: unique id broadcast + tlora_comm_create)


def grads_of(st):
    return {k: [t.clone() for s in range(len(l.ranks)) for t in l.read_grad(s)]
            for k, l in st.layers.items()}


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = Workload("dp-mini", [("q", 512, 768), ("k", 512, 256), ("o", 768, 512)],
                  [Job("a", 8, 2, 256), Job("b", 64, 3, 192), Job("c", 16, 1, 320)],
                  layers=2, seed=31)
    comm = bench.make_comm(local, rank, world)
    dp = TrainingStep(wl, device=local, nano_fixed=2, graphs=True, comm=comm)
    dp.init_random(wl.seed + rank)          # this replica's own inputs (seed + rank)
    solo = TrainingStep(wl, device=local, nano_fixed=2, graphs=True)
    solo.init_random(wl.seed + rank)
    # identical weights on every replica (overwrite the per-rank ones)
    ok = True
    fails = []

    def check(cond, what):
        nonlocal ok
        if not cond:
            ok = False
            fails.append(what)
    g0 = torch.Generator(device="cuda").manual_seed(999)
    for key in dp.keys:
        ld, ls = dp.layers[key], solo.layers[key]
        W = (torch.randn(ld.d, ld.k, generator=g0, device="cuda") * ld.d ** -0.5).bfloat16()
        ld.set_base(W)
        ls.set_base(W)
        for s, r in enumerate(ld.ranks):
            A = (torch.randn(ld.d, r, generator=g0, device="cuda") * ld.d ** -0.5)
            B = (torch.randn(r, ld.k, generator=g0, device="cuda") * r ** -0.5)
            ld.set_adapter(s, A, B)
            ls.set_adapter(s, A, B)
    for obj in (dp, solo):
        obj.enable_optimizer(1e-3, 0.01)
    solo.run()
    local_g = grads_of(solo)
    s1 = dp.run()
    got = grads_of(dp)
    for key in dp.keys:
        for a, b in zip(local_g[key], got[key]):
            ref = a.clone()
            dist.all_reduce(ref)  # NCCL sum of the local gradients, as the executor's comm
            scale = max(1.0, ref.abs().max().item())
            check(bool(torch.equal(ref, b)) if world == 2 else
                  (ref - b).abs().max().item() <= 1e-5 * scale, f"allreduce {key}")
    dp.run()
    for key in dp.keys:
        P = [t.clone() for s in range(len(dp.layers[key].ranks)) for t in dp.layers[key].read_adapter(s)]
        for t in P:
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t)
            check(all(torch.equal(parts[0], p) for p in parts), f"replicas {key}")
    check(s1.nano_used == 2, "nano")
    # ---- sharded optimizer: reduce-scatter -> AdamW on this rank's packed-row shard ->
    # all-gather of the bf16 operands; the same two steps from the same start state
    sh = TrainingStep(wl, device=local, nano_fixed=2, graphs=True, comm=comm, sharded_opt=True)
    sh.init_random(wl.seed + rank)
    g0 = torch.Generator(device="cuda").manual_seed(999)
    for key in sh.keys:
        ls = sh.layers[key]
        W = (torch.randn(ls.d, ls.k, generator=g0, device="cuda") * ls.d ** -0.5).bfloat16()
        ls.set_base(W)
        for s, r in enumerate(ls.ranks):
            ls.set_adapter(s, torch.randn(ls.d, r, generator=g0, device="cuda") * ls.d ** -0.5,
                           torch.randn(r, ls.k, generator=g0, device="cuda") * r ** -0.5)
    sh.enable_optimizer(1e-3, 0.01)
    sh.run()
    sh.run()
    torch.cuda.synchronize()
    # step 2's forward read the adapters step 1 refreshed: Y equal => the all-gathered bf16
    # operands equal the all-reduce path's (bitwise at 2 ranks, where a + b is exact-order)
    # (beyond 2 ranks the reduce-scatter and the all-reduce may sum in different orders; a
    # first Adam step then flips the sign of near-zero-gradient updates: |diff| <= 2 lr)
    for name in sh.names:
        a, b = sh.Y[name], dp.Y[name]
        if world == 2:
            check(bool(torch.equal(a, b)), f"Y {name}")
    # masters of the rows this rank owns == the all-reduce path's masters
    import ctypes as C
    from paper_2602_07263_b200 import capi
    for key in sh.keys:
        lay = sh.layers[key]
        lo, hi = C.c_int64(), C.c_int64()
        capi.call("tlora_layer_dp_shard", lay._h, comm, capi.GROUP_DP, C.byref(lo), C.byref(hi))
        for s in range(len(lay.ranks)):
            o, r = lay.offsets[s], lay.ranks[s]
            cols = [c for c in range(r) if lo.value <= o + c < hi.value]
            if not cols:
                continue
            Ash, Bsh = lay.read_adapter(s)
            Aar, Bar = dp.layers[key].read_adapter(s)
            idx = torch.tensor(cols, device="cuda")
            if world == 2:
                check(bool(torch.equal(Ash[:, idx], Aar[:, idx]) and torch.equal(Bsh[idx], Bar[idx])),
                      f"masters {key} {s}")
            else:
                lr = 1e-3 * (1.0 + 0.25 * (s % 4))
                dA = (Ash[:, idx] - Aar[:, idx]).abs()
                dB = (Bsh[idx] - Bar[idx]).abs()
                check(dA.max().item() <= 2.0001 * lr and dB.max().item() <= 2.0001 * lr,
                      f"masters {key} {s}")
                check((dA > 0.5 * lr).float().mean().item() < 0.01, f"flips {key} {s}")
    sh.close()
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(("STEP_DP_CHECK PASS" if flag.item() == 1 else "STEP_DP_CHECK FAIL") + f" world={world}",
              flush=True)
    if fails:
        print(f"rank {rank} failed checks: {fails[:8]}", flush=True)
    dp.close()
    solo.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
