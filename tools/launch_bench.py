"""Per-launch microbenchmark of one C2 projection (CUDA events, inputs resident).

  TLORA_LIB=<variant .so> python tools/launch_bench.py [proj]
Prints us/launch and achieved TFLOP/s or GB/s (algorithmic) for each of the six launches.
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_07263_b200.layer import FusedLoRALayer  # noqa: E402
from paper_2602_07263_b200.workload import config  # noqa: E402


def main():
    proj = sys.argv[1] if len(sys.argv) > 1 else "q"
    wl = config("C2")
    if proj == "all":
        for p in wl.projections:
            sys.argv[1:] = [p[0]]
            main()
        return
    name, d, k = [p for p in wl.projections if p[0] == proj][0]
    g = torch.Generator(device="cuda").manual_seed(0)
    lay = FusedLoRALayer(d, k, wl.ranks)
    lay.set_base((torch.randn(d, k, generator=g, device="cuda") * d ** -0.5).bfloat16())
    for s, r in enumerate(wl.ranks):
        lay.set_adapter(s, (torch.randn(d, r, generator=g, device="cuda") * d ** -0.5).bfloat16(),
                        (torch.randn(r, k, generator=g, device="cuda") * r ** -0.5).bfloat16())
    T = wl.tokens
    X = torch.randn(T, d, generator=g, device="cuda").bfloat16()
    dY = torch.randn(T, k, generator=g, device="cuda").bfloat16()
    plan = lay.plan(wl.token_slots())
    H = torch.empty(T, lay.R, dtype=torch.bfloat16, device="cuda")
    dH = torch.empty_like(H)
    Y = torch.empty(T, k, dtype=torch.bfloat16, device="cuda")
    dX = torch.empty(T, d, dtype=torch.bfloat16, device="cuda")
    rt = sum(j.tokens * j.rank for j in wl.jobs)
    ops = {
        "shrink": (lambda: lay.shrink(plan, X, H), 2 * (T * d + T * lay.R), "GB/s"),
        "fwd": (lambda: lay.fused_gemm(plan, X, H, Y), 2.0 * T * d * k + 2.0 * rt * k, "TF/s"),
        "dH": (lambda: lay.dh(plan, dY, dH), 2 * (T * k + T * lay.R), "GB/s"),
        "dX": (lambda: lay.dx(plan, dY, dH, dX), 2.0 * T * d * k + 2.0 * rt * d, "TF/s"),
        "dB": (lambda: lay.grad_b(plan, H, dY), 2 * (T * k + T * lay.R) + 4 * lay.R * k, "GB/s"),
        "dA": (lambda: lay.grad_a(plan, X, dH), 2 * (T * d + T * lay.R) + 4 * lay.R * d, "GB/s"),
        "dB+dA": (lambda: lay.grads(plan, H, dY, X, dH),
                  2 * (T * (d + k) + 2 * T * lay.R) + 4 * lay.R * (d + k), "GB/s"),
        "adamw": (lambda: lay.optimizer_step(), 32 * lay.R * (d + k), "GB/s"),
    }
    lay.set_optimizer(1e-4)
    lay.shrink(plan, X, H)
    lay.dh(plan, dY, dH)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = []
    for key, (fn, work, unit) in ops.items():
        for _ in range(3):
            fn()
        times = []
        for _ in range(20):
            flush.zero_()  # evict L2 between launches
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1e3)
        times.sort()
        us = times[len(times) // 2]
        rate = work / (us * 1e-6) / (1e12 if unit == "TF/s" else 1e9)
        out.append(f"{key}={us:.1f}us/{rate:.0f}{unit}")
    print(proj, " ".join(out), flush=True)


if __name__ == "__main__":
    main()
