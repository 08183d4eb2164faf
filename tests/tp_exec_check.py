"""The C++ tensor-parallel step (tlora_tp_*) vs round 1's Python TP driver (torchrun,
>= 2 GPUs; tests/test_gpu_executor.py). Same seeds, same shards, same nano-batch map and
the same deterministic boundary traffic (copy-engine all-gathers, slot-sum reduce-
scatters, the row-parallel reduce-scatter fused into the GEMM epilogue): one training step
of each, then every output this rank holds (column Y, row Y shard, dX shards) and every
adapter gradient / updated adapter are compared — bitwise for the activations, within
fp32 reassociation for the gradients (the replicated halves' NCCL all-reduce may pick a
different algorithm on the two communicators)."""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2602_07263_b200.tp import TPLayerSetStep  # noqa: E402
from paper_2602_07263_b200.tp_step import TPExecutor  # noqa: E402
from paper_2602_07263_b200.workload import config  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = config(os.environ.get("TP_CONFIG", "C2"))
    nano = int(os.environ.get("TP_NANO", "3"))
    py = TPLayerSetStep(wl, rank, world, local, nano=nano, fused_rs=True)
    py.enable_optimizer()
    comm = bench.make_comm(local, rank, world, tp_size=world)
    ex = TPExecutor(wl, rank, world, local, comm, nano_fixed=nano, fused_rs=True, copy_engine=True)
    ex.enable_optimizer()
    py.step(nano)
    s = ex.run()
    torch.cuda.synchronize()
    fails, worst = [], 0.0
    pairs = [(f"Y {n}", py.Y[n], ex.Y[n]) for n in ex.Y]
    pairs += [(f"Yshard {n}", py.Y_shard[n], ex.Y_shard[n]) for n in ex.Y_shard]
    pairs += [(f"dXloc {n}", py.dX_loc[n], ex.dX_loc[n]) for n in ex.dX_loc]
    pairs += [(f"dXshard {g}", py.dX_shard[g], ex.dX_shard[g]) for g in ex.dX_shard]
    for what, a, b in pairs:
        if not torch.equal(a, b):
            fails.append(what)
    for name, lay in ex.layers.items():
        for sl in range(len(wl.jobs)):
            for kind, ga, gb in zip(("dA", "dB", "A", "B"),
                                    py.layers[name].read_grad(sl) + py.layers[name].read_adapter(sl),
                                    lay.read_grad(sl) + lay.read_adapter(sl)):
                scale = max(1.0, ga.abs().max().item())
                err = (ga - gb).abs().max().item() / scale
                if kind in ("A", "B"):  # a first Adam step: reassociation may flip a sign
                    lr = 1e-4 * (1.0 + 0.25 * (sl % 4))
                    err = (ga - gb).abs().max().item()
                    if err > 2.0001 * lr:
                        fails.append(f"{kind} {name} {sl}")
                    continue
                worst = max(worst, err)
                if err > 1e-5:
                    fails.append(f"{kind} {name} {sl} {err:.2e}")
    ok = torch.tensor([0 if fails else 1], device="cuda")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if fails:
        print(f"rank{rank} mismatches: {fails[:10]}", flush=True)
    if rank == 0:
        print("TP_EXEC_CHECK", "PASS" if ok.item() == 1 else "FAIL",
              f"world={world} nano={s.nano_used} worst_grad_rel={worst:.2e}", flush=True)
    ex.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok.item() == 1 else 1)


if __name__ == "__main__":
    main()
