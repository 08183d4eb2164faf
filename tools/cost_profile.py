"""Measured B200 cost profile for the reference's planner.

The reference plans with analytic constants (proj/include/lora_fleet/hardware.hpp:7-25:
gpu_flops, kernel_launch_overhead, ...) and adapter_flops_per_token
(fused_lora.hpp:173-176). This tool times the real fused layer on one B200 over a grid of
shapes and fits, per launch class,

    t = overhead + flops / F + bytes / BW

(F: effective FLOP rate of the tensor-bound fused GEMMs; BW: effective bandwidth of the
HBM-bound low-rank launches), then writes profiles/b200_cost_profile.json:
  * hardware_spec: values to put into the reference's HardwareSpec (gpu_flops = the
    sustained fused-GEMM rate, kernel_launch_overhead = measured per-launch fixed cost);
  * predict(): the fitted per-layer fwd+bwd(+AdamW) step-time model and its error on the
    measured grid.

  python tools/cost_profile.py
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2602_07263_b200 import capi  # noqa: E402
from paper_2602_07263_b200.layer import FusedLoRALayer  # noqa: E402
import ctypes as C  # noqa: E402


def measure(d, k, ranks, tokens_per_job, reps=10):
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(d + k)
    lay = FusedLoRALayer(d, k, ranks)
    lay.set_base((torch.randn(d, k, generator=g, device=dev) * d ** -0.5).bfloat16())
    for s, r in enumerate(ranks):
        lay.set_adapter(s, (torch.randn(d, r, generator=g, device=dev) * d ** -0.5).bfloat16(),
                        (torch.randn(r, k, generator=g, device=dev) * r ** -0.5).bfloat16())
    lay.set_optimizer(1e-4)
    slots = np.repeat(np.arange(len(ranks)), tokens_per_job).astype(np.int32)
    T = len(slots)
    plan = lay.plan(slots)
    X = torch.randn(T, d, generator=g, device=dev).bfloat16()
    dY = torch.randn(T, k, generator=g, device=dev).bfloat16()
    Y = torch.empty(T, k, dtype=torch.bfloat16, device=dev)
    H = torch.zeros(T, lay.R, dtype=torch.bfloat16, device=dev)
    dX = torch.empty(T, d, dtype=torch.bfloat16, device=dev)

    def step():
        lay.forward(plan, X, Y, H)
        lay.backward(plan, dY, X, H, dX)
        lay.optimizer_step()

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    # step time WITHOUT the per-launch event brackets (they add a fixed cost per launch)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / reps
    # component times: every launch bracketed by CUDA events
    capi.call("tlora_profile_begin")
    for _ in range(reps):
        step()
    torch.cuda.synchronize()
    cnt, ms6, fl6 = (C.c_int32 * 6)(), (C.c_double * 6)(), (C.c_double * 6)()
    capi.call("tlora_profile_end", cnt, ms6, fl6)
    rt = sum(r * tokens_per_job for r in ranks)
    R = lay.R
    rec = {"d": d, "k": k, "T": T, "jobs": len(ranks), "ranks": list(ranks),
           "step_ms": step_ms,
           "gemm_ms": (ms6[capi.L_FWD] + ms6[capi.L_DX]) / reps,
           "gemm_flops": (fl6[capi.L_FWD] + fl6[capi.L_DX]) / reps,
           "lowrank_ms": sum(ms6[i] for i in (capi.L_SHRINK, capi.L_DH, capi.L_DB, capi.L_DA)) / reps,
           "lowrank_bytes": 2.0 * (2 * T * d + 2 * T * k + 4 * T * R) + 4.0 * R * (d + k),
           "optimizer_bytes": 32.0 * R * (d + k),
           "launches": int(sum(cnt)) / reps,
           "tok_rank": rt}
    lay.close()
    return rec


def fit(grid):
    """Model v2 (include/lora_fleet/hardware.hpp):
        step = fixed + gemm_flops / F + lowrank_bytes / BW + optimizer_bytes / BW_opt
    F and BW: slopes of the event-bracketed fused-GEMM (fwd + dX) and low-rank launch times;
    fixed and BW_opt: least squares of the unbracketed step time minus those two terms."""
    A = np.array([[2.0, r["gemm_flops"]] for r in grid])
    y = np.array([r["gemm_ms"] * 1e-3 for r in grid])
    (_, g_inv), *_ = np.linalg.lstsq(A, y, rcond=None)
    A2 = np.array([[3.0, r["lowrank_bytes"]] for r in grid])
    y2 = np.array([r["lowrank_ms"] * 1e-3 for r in grid])
    (_, l_inv), *_ = np.linalg.lstsq(A2, y2, rcond=None)
    rest = np.array([r["step_ms"] * 1e-3 - r["gemm_flops"] * g_inv - r["lowrank_bytes"] * l_inv
                     for r in grid])
    A3 = np.array([[1.0, r["optimizer_bytes"]] for r in grid])
    (fixed, o_inv), *_ = np.linalg.lstsq(A3, rest, rcond=None)
    F, BW, BWo = 1.0 / g_inv, 1.0 / l_inv, 1.0 / o_inv

    def predict(r):
        return fixed + r["gemm_flops"] / F + r["lowrank_bytes"] / BW + r["optimizer_bytes"] / BWo

    errs = [abs(predict(r) - r["step_ms"] * 1e-3) / (r["step_ms"] * 1e-3) for r in grid]
    return {
        "model_version": 2,
        "model": "step_s = fixed_overhead_s + gemm_flops/F + lowrank_bytes/BW + "
                 "optimizer_bytes/optimizer_BW",
        "F_flops_per_s": F, "BW_bytes_per_s": BW, "optimizer_BW_bytes_per_s": BWo,
        "fixed_overhead_s": fixed,
        "fit_rel_err_median": float(np.median(errs)), "fit_rel_err_max": float(np.max(errs)),
        "hardware_spec": {  # drop-in values for proj/include/lora_fleet/hardware.hpp
            "gpu_flops": F, "kernel_launch_overhead": fixed, "weight_stream_bw": BW,
            "note": "gpu_flops = sustained fused base+LoRA GEMM rate under the 1 kW cap; "
                    "kernel_launch_overhead = fixed cost of one fused layer's training step "
                    "(its launches), per nano-batch as nano_pipeline.hpp:79 charges it"},
    }


def main():
    grid = []
    for d, k in ((1024, 1024), (2048, 2048), (4096, 1024), (4096, 4096), (4096, 12288), (12288, 4096)):
        for ranks in ((8, 16, 32, 64), (8, 16, 24, 32, 48, 64, 96, 128)):
            for tpj in (256, 1024, 2048):
                grid.append(measure(d, k, ranks, tpj))
                print(f"d={d} k={k} jobs={len(ranks)} T={grid[-1]['T']} "
                      f"step={grid[-1]['step_ms']:.3f} ms", flush=True)
    out = fit(grid)
    out["device"] = torch.cuda.get_device_name(0)
    out["grid"] = grid
    path = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "b200_cost_profile.json"
    path.write_text(json.dumps(out, indent=1))
    print(json.dumps({k: v for k, v in out.items() if k != "grid"}, indent=1))


if __name__ == "__main__":
    main()
