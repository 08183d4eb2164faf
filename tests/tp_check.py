"""Tensor-parallel parity check (run under torchrun with >= 2 GPUs, one rank per GPU).

Every rank runs one fwd+bwd step of the TP layer set (paper_2602_07263_b200/tp.py) and
compares its shards against the UNSHARDED layer computed on the same inputs by the
single-GPU path (itself parity-checked against the CPU oracle in test_gpu_parity.py).
Tolerance (bf16 operands, NCCL bf16 reduce-scatter sums): max-abs <= 2e-2 * max(1,|ref|)
and Frobenius <= 1e-2 * ||ref|| for Y, dX, dA, dB.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tests/tp_check.py
"""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_07263_b200.layer import FusedLoRALayer  # noqa: E402
from paper_2602_07263_b200.tp import COLUMN, TPLayerSetStep  # noqa: E402
from paper_2602_07263_b200.workload import INPUT_GROUP, config  # noqa: E402


def errs(got, ref):
    got, ref = got.float(), ref.float()
    m = (got - ref).abs().max().item() / max(1.0, ref.abs().max().item())
    f = ((got - ref).norm() / max(ref.norm(), 1e-30)).item()
    return m, f


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = config(os.environ.get("TP_CONFIG", "C2"))
    nano = int(os.environ.get("TP_NANO", "4"))
    fused = os.environ.get("TP_FUSED_RS", "0") == "1"
    st = TPLayerSetStep(wl, rank, world, local, nano=nano, fused_rs=fused)
    st.step()
    torch.cuda.synchronize()
    nb, _ = st.plans(nano)
    P = world

    def shard_rows_of(full, b):  # this rank's SP rows of nano b inside a global tensor
        r0, n = b.shard(rank, P)
        return full[b.t0 + r0:b.t0 + r0 + n]

    def gather_cols(t):
        parts = [torch.empty_like(t) for _ in range(P)]
        dist.all_gather(parts, t.contiguous())
        return torch.cat(parts, dim=1)

    slots = torch.cat([torch.from_numpy(b.slots) for b in nb]).numpy()
    worst = 0.0
    report = []
    dX_ref_group = {}
    for name, d, k in wl.projections:
        W, As, Bs = st.full_weights[name]
        ref = FusedLoRALayer(d, k, wl.ranks, device=local)
        ref.set_base(W)
        for s in range(len(wl.jobs)):
            ref.set_adapter(s, As[s], Bs[s])
        plan = ref.plan(slots)
        if name in COLUMN:
            X = st.X_full[INPUT_GROUP[name]]
            dY = gather_cols(st.dY[name])
        else:
            X = gather_cols(st.X_loc[name])
            dY = st.dY_full[name]
        Y, H = ref.forward(plan, X)
        dX = ref.backward(plan, dY, X, H)
        torch.cuda.synchronize()
        lay = st.layers[name]
        w = k // P if name in COLUMN else d // P
        checks = []
        if name in COLUMN:
            checks.append(("Y", st.Y[name], Y[:, rank * w:(rank + 1) * w]))
            g = INPUT_GROUP[name]
            dX_ref_group[g] = dX.float() if g not in dX_ref_group else dX_ref_group[g] + dX.float()
        else:
            ys = torch.cat([st._srows(st.Y_shard[name], b) for b in nb])
            yr = torch.cat([shard_rows_of(Y, b) for b in nb])
            checks.append(("Y", ys, yr))
            checks.append(("dX", st.dX_loc[name], dX[:, rank * (d // P):(rank + 1) * (d // P)]))
        for s in range(len(wl.jobs)):
            dA_ref, dB_ref = ref.read_grad(s)
            dA, dB = lay.read_grad(s)
            if name in COLUMN:
                checks.append((f"dA{s}", dA, dA_ref))
                checks.append((f"dB{s}", dB, dB_ref[:, rank * w:(rank + 1) * w]))
            else:
                checks.append((f"dA{s}", dA, dA_ref[rank * w:(rank + 1) * w]))
                checks.append((f"dB{s}", dB, dB_ref))
        for key, got, want in checks:
            m, f = errs(got, want)
            worst = max(worst, m)
            ok = m <= 2e-2 and f <= 1e-2
            report.append((name, key, m, f, ok))
        ref.close()
    for g, dXr in dX_ref_group.items():
        xs = torch.cat([st._srows(st.dX_shard[g], b) for b in nb])
        xr = torch.cat([shard_rows_of(dXr, b) for b in nb])
        m, f = errs(xs, xr)
        report.append((g, "dX", m, f, m <= 2e-2 and f <= 1e-2))
    bad = [r for r in report if not r[4]]
    ok = torch.tensor([0 if bad else 1], device="cuda")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if rank == 0 or bad:
        for r in report:
            if not r[4] or r[1] in ("Y", "dX"):
                print(f"rank{rank} {r[0]:5s} {r[1]:4s} maxrel={r[2]:.2e} frob={r[3]:.2e} "
                      f"{'ok' if r[4] else 'FAIL'}", flush=True)
    if rank == 0:
        print("TP_CHECK", "PASS" if ok.item() == 1 else "FAIL",
              f"world={world} nano={nano} fused_rs={fused}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok.item() == 1 else 1)


if __name__ == "__main__":
    main()
