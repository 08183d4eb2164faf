"""First-light GPU checks of the tcgen05 path against a torch fp32 restatement.

The oracle-based parity tests (tests/test_gpu_parity.py) are the gate; this file is a
fast diagnostic that isolates each of the six launches.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(X, W, As, Bs, slots):
    """fp32 restatement of fused_lora.hpp:84-119 on bf16-rounded inputs (+ backward)."""
    Xf, Wf = X.float(), W.float()
    Y = Xf @ Wf
    H = torch.zeros(X.shape[0], sum(((a.shape[1] + 7) // 8) * 8 for a in As), device=X.device)
    return Y, H


def _case(T, d, k, ranks, shuffle, seed=0):
    g = torch.Generator().manual_seed(seed)
    from paper_2602_07263_b200.layer import FusedLoRALayer
    S = len(ranks)
    counts = np.random.RandomState(seed).multinomial(T - S, [1.0 / S] * S) + 1
    slots = np.repeat(np.arange(S), counts).astype(np.int32)
    if shuffle:
        np.random.RandomState(seed + 1).shuffle(slots)
    X = torch.randn(T, d, generator=g).bfloat16().cuda()
    W = (torch.randn(d, k, generator=g) / d ** 0.5).bfloat16().cuda()
    As = [(torch.randn(d, r, generator=g) / d ** 0.5).bfloat16().cuda() for r in ranks]
    Bs = [(torch.randn(r, k, generator=g) / r ** 0.5).bfloat16().cuda() for r in ranks]
    dY = torch.randn(T, k, generator=g).bfloat16().cuda()
    lay = FusedLoRALayer(d, k, ranks)
    lay.set_base(W)
    for s in range(S):
        lay.set_adapter(s, As[s], Bs[s])
    plan = lay.plan(slots)
    Y, H = lay.forward(plan, X, y_dtype=torch.float32)
    dX = lay.backward(plan, dY, X, H)
    torch.cuda.synchronize()
    # fp32 reference
    st = torch.from_numpy(slots).long().cuda()
    Xf, Wf, dYf = X.float(), W.float(), dY.float()
    Yr = Xf @ Wf
    dXr = dYf @ Wf.t()
    errs = {}
    for s in range(S):
        idx = (st == s).nonzero().flatten()
        if idx.numel() == 0:
            continue
        A, B = As[s].float(), Bs[s].float()
        h = (Xf[idx] @ A)
        hb = h.bfloat16().float()
        Yr[idx] += hb @ B
        dh = (dYf[idx] @ B.t())
        dhb = dh.bfloat16().float()
        dXr[idx] += dhb @ A.t()
        off, r = lay.offsets[s], ranks[s]
        hk = H[idx, off:off + r].float()
        errs[f"H{s}"] = ((hk - h).norm() / h.norm()).item()
        dA, dB = lay.read_grad(s)
        dAr = Xf[idx].t() @ dhb
        dBr = hb.t() @ dYf[idx]
        errs[f"dA{s}"] = ((dA - dAr).norm() / dAr.norm()).item()
        errs[f"dB{s}"] = ((dB - dBr).norm() / dBr.norm()).item()
    errs["Y"] = ((Y - Yr).norm() / Yr.norm()).item()
    errs["dX"] = ((dX.float() - dXr).norm() / dXr.norm()).item()
    return errs


@pytest.mark.parametrize("T,d,k,ranks,shuffle", [
    (256, 128, 256, [16], False),
    (1000, 512, 768, [8, 16, 32, 64], False),
    (777, 256, 264, [8, 24, 128], True),
    (4096, 1024, 1024, [8, 16, 32, 64], True),
])
def test_fwd_bwd_vs_torch(T, d, k, ranks, shuffle):
    errs = _case(T, d, k, ranks, shuffle)
    print(errs)
    for key, e in errs.items():
        assert e < 1e-2, (key, e, errs)
