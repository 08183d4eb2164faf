"""Per-shape fused base+LoRA GEMM (lora_gemm2_kernel) vs cuBLAS base GEMM on one B200.

For every C2 projection: our fused forward (Y = XW + H·Bcat over the packed-rank window)
and fused dX, against torch.matmul (cuBLAS) of the base product alone, interleaved in
rounds so clock / power drift hits both arms alike. TFLOP/s are algorithmic: base
2·T·d·k (+ the LoRA expand FLOPs for ours).

  python tools/gemm_vs_cublas.py [C2] [--rounds 5] [--reps 10]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2602_07263_b200.layer import FusedLoRALayer  # noqa: E402
from paper_2602_07263_b200.workload import config  # noqa: E402


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C2")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    wl = config(args.config)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(1)
    slots = wl.token_slots()
    T = len(slots)
    rt = sum(j.tokens * j.rank for j in wl.jobs)
    out = []
    for name, d, k in wl.projections:
        if args.only and name not in args.only.split(","):
            continue
        lay = FusedLoRALayer(d, k, wl.ranks)
        W = (torch.randn(d, k, generator=g, device=dev) * d ** -0.5).bfloat16()
        lay.set_base(W)
        for s, j in enumerate(wl.jobs):
            lay.set_adapter(s, (torch.randn(d, j.rank, generator=g, device=dev) * 0.02).bfloat16(),
                            (torch.randn(j.rank, k, generator=g, device=dev) * 0.02).bfloat16())
        plan = lay.plan(slots)
        X = torch.randn(T, d, generator=g, device=dev).bfloat16()
        dY = torch.randn(T, k, generator=g, device=dev).bfloat16()
        H = torch.zeros(T, lay.R, dtype=torch.bfloat16, device=dev)
        dH = torch.zeros(T, lay.R, dtype=torch.bfloat16, device=dev)
        lay.shrink(plan, X, H)
        lay.dh(plan, dY, dH)
        Y = torch.empty(T, k, dtype=torch.bfloat16, device=dev)
        dX = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
        Wt = W.t()
        arms = {
            "ours_fwd": lambda: lay.fused_gemm(plan, X, H, Y),
            "cublas_fwd": lambda: torch.matmul(X, W, out=Y),
            "ours_dx": lambda: lay.dx(plan, dY, dH, dX),
            "cublas_dx": lambda: torch.matmul(dY, Wt, out=dX),
        }
        for fn in arms.values():
            for _ in range(3):
                fn()
        torch.cuda.synchronize()
        ms = {a: [] for a in arms}
        for _ in range(args.rounds):
            for a, fn in arms.items():
                ms[a].append(timed(fn, args.reps))
        base = 2.0 * T * d * k
        rec = {"proj": name, "d": d, "k": k, "T": T}
        for a in arms:
            best = min(ms[a])
            med = sorted(ms[a])[len(ms[a]) // 2]
            fl = base + (2.0 * rt * (k if a == "ours_fwd" else d) if a.startswith("ours") else 0.0)
            rec[a] = {"ms_med": round(med, 4), "tflops_med": round(fl / med / 1e9, 1),
                      "tflops_best": round(fl / best / 1e9, 1)}
        out.append(rec)
        print(json.dumps(rec), flush=True)
        lay.close()
        del X, dY, H, dH, Y, dX, W
        torch.cuda.empty_cache()
    tot = {a: sum(r[a]["ms_med"] for r in out) for a in ("ours_fwd", "cublas_fwd", "ours_dx", "cublas_dx")}
    print(json.dumps({"total_ms_med": {a: round(v, 4) for a, v in tot.items()}}))


if __name__ == "__main__":
    main()
