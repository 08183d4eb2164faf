"""C5 heterogeneity sweep (BASELINE.json configs[4]): ranks 4-256, 2-32 jobs, Zipf(1.2)-
skewed batches, d = k in {1024, 4096}, T in {2048, 8192}. Per cell: GPU training-step
throughput (fwd + bwd + AdamW through the C-ABI, CUDA events), rank-packing efficiency of
the plan, and — for the T = 2048 cells — parity against the double CPU oracle (with
bf16-emulated intermediates) plus the oracle's own fwd+bwd time on the host cores.

  python tools/c5_sweep.py [--seeds 5] > profiles/r1_c5_sweep.md
"""
import argparse
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as O  # noqa: E402  (checker only)

from paper_2602_07263_b200.layer import FusedLoRALayer  # noqa: E402
from paper_2602_07263_b200.workload import c5_cell  # noqa: E402


def run_cell(d, J, T, seed, check):
    wl = c5_cell(d, J, T, seed)
    rs = np.random.RandomState(seed)
    ranks = wl.ranks
    slots = wl.token_slots()
    bf = O.round_bf16
    X = bf(rs.randn(T, d))
    W = bf(rs.randn(d, d) / np.sqrt(d))
    A = [bf(rs.randn(d, r) / np.sqrt(d)) for r in ranks]
    B = [bf(rs.randn(r, d) / np.sqrt(r)) for r in ranks]
    dY = bf(rs.randn(T, d))
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev).bfloat16()  # noqa: E731
    lay = FusedLoRALayer(d, d, ranks)
    lay.set_base(t(W))
    for s in range(J):
        lay.set_adapter(s, t(A[s]), t(B[s]))
    lay.set_optimizer(1e-4, 0.0)
    plan = lay.plan(slots)
    info = plan.info()
    Xd, dYd = t(X), t(dY)
    Y = torch.empty(T, d, dtype=torch.float32, device=dev)
    H = torch.zeros(T, lay.R, dtype=torch.bfloat16, device=dev)
    dX = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
    out = {"d": d, "J": J, "T": T, "seed": seed, "rmin": min(ranks), "rmax": max(ranks),
           "pack": info.useful_ext_cols / max(1, info.packed_ext_cols)}
    if check:  # parity before any optimizer step changes the adapters
        lay.forward(plan, Xd, Y, H)
        lay.backward(plan, dYd, Xd, H, dX)
        torch.cuda.synchronize()
        Ye = O.fused_forward(X, W, A, B, slots, round_bf16=True)
        t0 = time.perf_counter()
        O.fused_forward(X, W, A, B, slots)
        dXe, dAe, dBe = O.fused_backward(X, W, A, B, slots, dY)
        out["cpu_s"] = time.perf_counter() - t0
        rel = lambda a, b: float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))  # noqa: E731
        out["errY"] = rel(Y.double().cpu().numpy(), Ye)
        out["errdX"] = rel(dX.double().cpu().numpy(), dXe)
        out["errG"] = max(max(rel(g.double().cpu().numpy(), e) for g, e in zip(lay.read_grad(s), (dAe[s], dBe[s])))
                          for s in range(J))
    bf16_out = torch.empty(T, d, dtype=torch.bfloat16, device=dev)

    def step():
        lay.forward(plan, Xd, bf16_out, H)
        lay.backward(plan, dYd, Xd, H, dX)
        lay.optimizer_step()

    for _ in range(3):
        step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    out["ms"] = ms
    out["tok_s"] = T / (ms / 1e3)
    rt = sum(j.tokens * j.rank for j in wl.jobs)
    out["tflops"] = (4.0 * T * d * d + 6.0 * rt * 2 * d) / (ms / 1e3) / 1e12
    lay.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=5)
    args = ap.parse_args()
    rows = []
    for d in (1024, 4096):
        for J in (2, 4, 8, 16, 32):
            for T in (2048, 8192):
                for seed in range(1, args.seeds + 1):
                    rows.append(run_cell(d, J, T, seed, check=(T == 2048)))
    print("# C5 heterogeneity sweep (one B200, training step = fwd + bwd + AdamW)\n")
    print(f"{len(rows)} cells; host threads for the oracle: {os.cpu_count()}. Parity columns are")
    print("max-abs / max(1,|ref|) vs the double oracle (plain, not bf16-emulated) on the same")
    print("bf16 inputs; bounds in tests/test_gpu_parity.py are 1e-2 (Y) and 2e-2 (dX, grads).\n")
    print("| d | jobs | T | seed | ranks | pack eff. | ms/step | tokens/s | TFLOP/s | "
          "err Y | err dX | err dA/dB | oracle fwd+bwd s |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        chk = (f"{r['errY']:.1e} | {r['errdX']:.1e} | {r['errG']:.1e} | {r['cpu_s']:.2f}"
               if "errY" in r else "— | — | — | —")
        print(f"| {r['d']} | {r['J']} | {r['T']} | {r['seed']} | {r['rmin']}–{r['rmax']} | "
              f"{r['pack']:.2f} | {r['ms']:.3f} | {r['tok_s']:,.0f} | {r['tflops']:.0f} | {chk} |")
    bad = [r for r in rows if "errY" in r and (r["errY"] > 1e-2 or r["errdX"] > 2e-2 or r["errG"] > 2e-2)]
    print(f"\nparity: {sum('errY' in r for r in rows) - len(bad)} / {sum('errY' in r for r in rows)} "
          f"checked cells within bounds")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
