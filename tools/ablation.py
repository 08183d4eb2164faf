"""Fused vs unfused multi-LoRA ablation on one B200.

The reference accounts for the unfused design analytically (unfused_cost,
proj/include/lora_fleet/fused_lora.hpp:139-163: +4 launches per active adapter and the
extra gather / scatter bytes). This tool runs that design for real, next to the fused
path, on the same workload (fwd + bwd of every projection, synthetic inputs):

  fused        this repo: LayerSetStep (tlora C-ABI kernels), CUDA graph replay
  unfused      cuBLAS (torch.matmul) base GEMM + per-job LoRA GEMMs, the reference's
               fused_forward structure (fused_lora.hpp:93-113) plus the matching backward:
               Y = XW; per job  H_j = X_j A_j,  Y_j += H_j B_j;  dX = dY Wᵀ; per job
               dH_j = dY_j B_jᵀ, dB_j = H_jᵀ dY_j, dA_j = X_jᵀ dH_j, dX_j += dH_j A_jᵀ
               (bf16 grads: cheaper than the fused path's fp32, so the baseline is favoured)
  base_only    cuBLAS Y = XW and dX = dY Wᵀ alone: the no-adapter floor

Torch arms are timed eager and as CUDA-graph replays (launch overhead removed; the
per-launch GPU ramp / tail of many small GEMMs remains, which is the unfused design's
real device-side cost). Tokens job-contiguous (views, no gather), again favouring the
baseline.

  python tools/ablation.py [C2] [--steps 20]  -> prints one JSON object
"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2602_07263_b200.runner import LayerSetStep  # noqa: E402
from paper_2602_07263_b200.workload import INPUT_GROUP, config  # noqa: E402


def time_fn(fn, steps, warmup=3, graph=False):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            fn()
        run = g.replay
        run()
    else:
        run = fn
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


class TorchArm:
    def __init__(self, wl, lora: bool, seed=2602):
        dev = torch.device("cuda", 0)
        g = torch.Generator(device=dev).manual_seed(seed)
        T = wl.tokens
        self.wl, self.lora = wl, lora
        self.bounds = []
        t0 = 0
        for j in wl.jobs:
            self.bounds.append((t0, t0 + j.tokens))
            t0 += j.tokens
        self.W, self.A, self.B, self.X, self.Y, self.dY, self.dX, self.H = {}, {}, {}, {}, {}, {}, {}, {}
        self.dA, self.dB, self.dH = {}, {}, {}
        for name, d, k in wl.projections:
            self.W[name] = (torch.randn(d, k, generator=g, device=dev) * d ** -0.5).bfloat16()
            self.A[name] = [(torch.randn(d, j.rank, generator=g, device=dev) * d ** -0.5).bfloat16()
                            for j in wl.jobs]
            self.B[name] = [(torch.randn(j.rank, k, generator=g, device=dev) * j.rank ** -0.5).bfloat16()
                            for j in wl.jobs]
            grp = INPUT_GROUP.get(name, name)
            if grp not in self.X:
                self.X[grp] = torch.randn(T, d, generator=g, device=dev).bfloat16()
            self.Y[name] = torch.empty(T, k, dtype=torch.bfloat16, device=dev)
            self.dY[name] = torch.randn(T, k, generator=g, device=dev).bfloat16()
            self.dX[name] = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
            self.H[name] = [torch.empty(e - s, j.rank, dtype=torch.bfloat16, device=dev)
                            for (s, e), j in zip(self.bounds, wl.jobs)]
            self.dH[name] = [torch.empty_like(h) for h in self.H[name]]
            self.dA[name] = [torch.empty_like(a) for a in self.A[name]]
            self.dB[name] = [torch.empty_like(b) for b in self.B[name]]

    def step(self):
        names = [p[0] for p in self.wl.projections]
        for name in names:
            X, Y = self.X[INPUT_GROUP.get(name, name)], self.Y[name]
            torch.matmul(X, self.W[name], out=Y)
            if self.lora:
                for i, (s, e) in enumerate(self.bounds):
                    torch.matmul(X[s:e], self.A[name][i], out=self.H[name][i])
                    Ys = Y[s:e]
                    Ys.addmm_(self.H[name][i], self.B[name][i])
        for name in reversed(names):
            X, dY, dX = self.X[INPUT_GROUP.get(name, name)], self.dY[name], self.dX[name]
            torch.matmul(dY, self.W[name].t(), out=dX)
            if self.lora:
                for i, (s, e) in enumerate(self.bounds):
                    dYs = dY[s:e]
                    torch.matmul(dYs, self.B[name][i].t(), out=self.dH[name][i])
                    torch.matmul(self.H[name][i].t(), dYs, out=self.dB[name][i])
                    torch.matmul(X[s:e].t(), self.dH[name][i], out=self.dA[name][i])
                    dX[s:e].addmm_(self.dH[name][i], self.A[name][i].t())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C2")
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    wl = config(args.config)
    T = wl.tokens
    out = {"config": wl.name, "tokens_per_step": T, "jobs": len(wl.jobs),
           "projections": len(wl.projections), "what": "fwd+bwd of every projection, no optimizer"}

    st = LayerSetStep(wl, device=0)
    from paper_2602_07263_b200 import capi
    n0 = capi.lib().tlora_launch_count()
    st.forward()
    st.backward()
    torch.cuda.synchronize()
    fused_launches = capi.lib().tlora_launch_count() - n0

    def fused():
        st.forward()
        st.backward()
    res = {"fused": {"eager_ms": time_fn(fused, args.steps),
                     "graph_ms": time_fn(fused, args.steps, graph=True),
                     "launches_per_step": fused_launches}}
    del st
    torch.cuda.empty_cache()
    for arm, lora in (("unfused", True), ("base_only", False)):
        ta = TorchArm(wl, lora)
        res[arm] = {"eager_ms": time_fn(ta.step, args.steps),
                    "graph_ms": time_fn(ta.step, args.steps, graph=True),
                    "launches_per_step": len(wl.projections) * (2 + (6 * len(wl.jobs) if lora else 0))}
        del ta
        torch.cuda.empty_cache()
    for arm in res.values():
        arm["tokens_per_s_graph"] = round(T / (arm["graph_ms"] / 1e3), 1)
        arm["tokens_per_s_eager"] = round(T / (arm["eager_ms"] / 1e3), 1)
        arm["graph_ms"] = round(arm["graph_ms"], 4)
        arm["eager_ms"] = round(arm["eager_ms"], 4)
    out["arms"] = res
    out["fused_speedup_vs_unfused_graph"] = round(res["unfused"]["graph_ms"] / res["fused"]["graph_ms"], 3)
    out["fused_speedup_vs_unfused_eager"] = round(res["unfused"]["eager_ms"] / res["fused"]["eager_ms"], 3)
    out["fused_vs_base_only_graph"] = round(res["base_only"]["graph_ms"] / res["fused"]["graph_ms"], 3)
    out["device"] = torch.cuda.get_device_name(0)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
