"""NVLink evidence for the fused GEMM + reduce-scatter (tlora_forward_gemm_rs) from ONE
process (ncu must not wrap a multi-rank command): rank 0's row-parallel C4 down-projection
forward at TP = world runs on GPU 0 and its epilogue bulk-copies every row owned by rank p
straight into GPU p's receive slot over NVLink (peer access enabled here, as torch's
symmetric memory does for the TP driver). Checks the slots against the plain fused GEMM.

  python tools/gemm_rs_nvlink.py --world 2
  ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum \
      -k regex:lora_gemm2 python tools/gemm_rs_nvlink.py --world 2
Expected NVLink payload of the launch: (world - 1) / world of the T x k bf16 output.
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2602_07263_b200.layer import FusedLoRALayer  # noqa: E402
from paper_2602_07263_b200.workload import config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--tokens", type=int, default=30720)  # C4 global batch / 2 nano-batches
    a = ap.parse_args()
    P = a.world
    assert torch.cuda.device_count() >= P, "needs one GPU per rank"
    from cuda import cudart
    torch.cuda.set_device(0)
    for p in range(1, P):
        err, ok = cudart.cudaDeviceCanAccessPeer(0, p)
        assert ok, f"GPU 0 cannot access GPU {p}"
        (err,) = cudart.cudaDeviceEnablePeerAccess(p, 0)
        assert int(err) in (0, 704), err  # 704 = already enabled
    wl = config("C4")
    _, d_full, k = [x for x in wl.projections if x[0] == "down"][0]
    d, T = d_full // P, a.tokens
    g = torch.Generator(device="cuda").manual_seed(5)
    lay = FusedLoRALayer(d, k, wl.ranks, device=0)
    lay.set_base((torch.randn(d, k, generator=g, device="cuda") * d ** -0.5).bfloat16())
    for s, r in enumerate(wl.ranks):
        lay.set_adapter(s, (torch.randn(d, r, generator=g, device="cuda") * d ** -0.5).bfloat16(),
                        (torch.randn(r, k, generator=g, device="cuda") * r ** -0.5).bfloat16())
    counts = np.full(len(wl.jobs), T // len(wl.jobs))
    counts[0] += T - counts.sum()
    plan = lay.plan(np.repeat(np.arange(len(wl.jobs)), counts).astype(np.int32))
    X = torch.randn(T, d, generator=g, device="cuda").bfloat16()
    H = torch.empty(T, lay.R, dtype=torch.bfloat16, device="cuda")
    lay.shrink(plan, X, H)
    rows = T // P
    recv = [torch.zeros(P, rows, k, dtype=torch.bfloat16, device=f"cuda:{p}") for p in range(P)]
    Y = torch.empty(T, k, dtype=torch.bfloat16, device="cuda")
    lay.fused_gemm(plan, X, H, Y)
    for _ in range(2):
        lay.fused_gemm_rs(plan, X, H, [t.data_ptr() for t in recv], 0, rows, 0)
    for p in range(P):
        torch.cuda.synchronize(p)
    ok = all(torch.equal(recv[p][0].to("cuda:0"), Y[p * rows:(p + 1) * rows]) for p in range(P))
    peer_bytes = (P - 1) * rows * k * 2
    print(f"gemm_rs TP{P}: down {d}x{k}, T={T}: slots {'OK' if ok else 'MISMATCH'}; "
          f"expected NVLink payload per launch {peer_bytes / 1e6:.1f} MB")
    if not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
