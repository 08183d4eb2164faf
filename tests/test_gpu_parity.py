"""GPU parity: the sm_100a path (through the C-ABI) vs the oracle on the same inputs.

Tolerances (stated per SURVEY.md §8(c)); all comparisons are on the SAME bf16-rounded
inputs the device sees:
  * vs the double oracle with bf16-emulated intermediates (H, dH rounded like the device):
      Y (fp32 out)   max-abs <= 3e-3 * max(1, max|ref|)   (a near-tie of the fp32-vs-double
                     H value can round to the neighbouring bf16: 1 ulp of H times |B|)
      dX (bf16 out)  max-abs <= 8e-3 * max(1, max|ref|)    (one bf16 output rounding)
      dA, dB (fp32)  ||diff||_F <= 2e-3 * ||ref||_F
  * vs the plain double oracle (reference semantics, no emulation):
      Y              max-abs <= 1e-2 * max(1, max|ref|), ||diff||_F <= 4e-3 * ||ref||_F
      dX, dA, dB     max-abs <= 2e-2 * max(1, max|ref|), ||diff||_F <= 8e-3 * ||ref||_F
      (dX, dA carry the bf16 rounding of dH = dY·Bᵀ, which dominates when the adapter
       term outweighs the base term, as in the reference's N(0,1) test instances)
  * the reference's own golden outputs on the ORIGINAL double inputs (so the bound also
    absorbs bf16 input quantisation): Y max-abs <= 2e-2 * max(1, max|ref|),
    ||diff||_F <= 1e-2 * ||ref||_F.
Bit-exact properties at full size: Y(2X) == 2 Y(X), permutation equivariance of Y.
"""
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
import oracle as O  # noqa: E402
from golden_io import read_records  # noqa: E402

from paper_2602_07263_b200.layer import FusedLoRALayer  # noqa: E402
from paper_2602_07263_b200.workload import c5_cell, config  # noqa: E402

pytestmark = pytest.mark.gpu


def pad8(n):
    return (n + 7) // 8 * 8


def bf(a):
    return O.round_bf16(np.asarray(a, np.float64))


def gpu_run(X, W, A, B, slots, dY, beta_runs=1, gathered=False):
    """Run fwd+bwd through the C-ABI on padded bf16 copies; returns numpy results.
    gathered: tlora_plan_create_gathered + tlora_gather_rows (operands in job-sorted order,
    Y / dX stored back in token order by the epilogues; H un-gathered here for the check)."""
    T, d = X.shape
    k = W.shape[1]
    dp, kp = pad8(d), pad8(k)
    ranks = [a.shape[1] for a in A]
    dev = torch.device("cuda", 0)

    def padded(a, rows, cols):
        out = np.zeros((rows, cols))
        out[: a.shape[0], : a.shape[1]] = a
        return torch.from_numpy(out).to(dev).bfloat16()

    lay = FusedLoRALayer(dp, kp, ranks)
    lay.set_base(padded(W, dp, kp))
    for s in range(len(A)):
        lay.set_adapter(s, padded(A[s], dp, ranks[s]), padded(B[s], ranks[s], kp))
    plan = lay.plan(slots, gathered=gathered)
    Xd = padded(X, T, dp)
    dYd = padded(dY, T, kp)
    if gathered:
        Xg, dYg = torch.empty_like(Xd), torch.empty_like(dYd)
        plan.gather([(Xd, Xg), (dYd, dYg)])
        Xd, dYd = Xg, dYg
    Y, H = lay.forward(plan, Xd, y_dtype=torch.float32)
    dX = None
    for i in range(beta_runs):
        dX = lay.backward(plan, dYd, Xd, H, beta=1.0 if i else 0.0)
    torch.cuda.synchronize()
    if gathered:
        Hn = torch.empty_like(H)
        Hn[torch.from_numpy(plan.row_map().astype(np.int64)).to(dev)] = H
        H = Hn
    grads = [lay.read_grad(s) for s in range(len(A))]
    out = dict(Y=Y[:, :k].double().cpu().numpy(), dX=dX[:, :d].double().cpu().numpy(),
               dA=[g[0][:d].double().cpu().numpy() for g in grads],
               dB=[g[1][:, :k].double().cpu().numpy() for g in grads],
               H=H.double().cpu().numpy(), offsets=lay.offsets, plan=plan.info())
    lay.close()
    return out


def maxrel(a, b):
    return np.abs(a - b).max() / max(1.0, np.abs(b).max())


def frob(a, b):
    n = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (n if n > 0 else 1.0)


def check(got, X, W, A, B, slots, dY, scale_grads=1.0):
    Ye, He = O.fused_forward(X, W, A, B, slots, round_bf16=True, want_h=True)
    dXe, dAe, dBe = O.fused_backward(X, W, A, B, slots, dY, round_bf16=True)
    assert maxrel(got["Y"], Ye) <= 3e-3, maxrel(got["Y"], Ye)
    assert maxrel(got["dX"], dXe) <= 8e-3, maxrel(got["dX"], dXe)
    for s in range(len(A)):
        if not np.any(slots == s):
            assert not np.any(got["dA"][s]) and not np.any(got["dB"][s])
            continue
        assert frob(got["dA"][s], scale_grads * dAe[s]) <= 2e-3, (s, frob(got["dA"][s], dAe[s]))
        assert frob(got["dB"][s], scale_grads * dBe[s]) <= 2e-3, (s, frob(got["dB"][s], dBe[s]))
    # plain double oracle (reference semantics)
    Yp = O.fused_forward(X, W, A, B, slots)
    dXp, dAp, dBp = O.fused_backward(X, W, A, B, slots, dY)
    assert maxrel(got["Y"], Yp) <= 1e-2 and frob(got["Y"], Yp) <= 4e-3
    assert maxrel(got["dX"], dXp) <= 2e-2 and frob(got["dX"], dXp) <= 8e-3
    for s in range(len(A)):
        if np.any(slots == s):
            assert maxrel(got["dA"][s], scale_grads * dAp[s]) <= 2e-2
            assert frob(got["dA"][s], scale_grads * dAp[s]) <= 8e-3
            assert maxrel(got["dB"][s], scale_grads * dBp[s]) <= 2e-2
            assert frob(got["dB"][s], scale_grads * dBp[s]) <= 8e-3
    # the stashed H is exactly the masked per-token intermediate
    Hg = got["H"]
    for s in range(len(A)):
        rows = np.where(slots == s)[0]
        if rows.size == 0:
            continue
        o, r = got["offsets"][s], A[s].shape[1]
        he = He[rows][:, sum(a.shape[1] for a in A[:s]):sum(a.shape[1] for a in A[:s + 1])]
        assert maxrel(Hg[rows, o:o + r], he) <= 1e-2
        mask = np.ones(Hg.shape[1], bool)
        mask[o:o + r] = False
        assert not np.any(Hg[np.ix_(rows, np.where(mask)[0])]), "H not masked to own columns"


def golden_cases(name, n):
    insts = read_records((ROOT / "tests" / "golden" / name).read_bytes())[:n]
    out = []
    for inst in insts:
        order = inst.slot_order()
        pos = {a: s for s, a in enumerate(order)}
        slots = np.array([pos[a] for a in inst.owner], np.int32)
        out.append((inst, [inst.A[a] for a in order], [inst.B[a] for a in order], slots))
    return out


@pytest.mark.parametrize("name,n,gathered", [("fused_2024.bin", 50, False),
                                             ("fused_101.bin", 25, False),
                                             ("fused_2024.bin", 50, True)])
def test_reference_golden_instances(name, n, gathered):
    for inst, A, B, slots in golden_cases(name, n):
        X, W = bf(inst.X), bf(inst.W)
        Ab, Bb = [bf(a) for a in A], [bf(b) for b in B]
        dY = bf(np.random.RandomState(inst.tokens).randn(inst.tokens, inst.k))
        got = gpu_run(X, W, Ab, Bb, slots, dY, gathered=gathered)
        check(got, X, W, Ab, Bb, slots, dY)
        # against the reference's own output on the original double inputs
        assert maxrel(got["Y"], inst.Y_fused) <= 2e-2
        assert frob(got["Y"], inst.Y_fused) <= 1e-2


def test_kat_exact():
    W = np.array([[1, 0], [0, 1], [1, 1]], float)
    A = np.array([[1], [0], [0]], float)
    B = np.array([[2, 3]], float)
    X = np.array([[1, 2, 3], [0, 1, 0]], float)
    got = gpu_run(X, W, [A], [B], np.array([0, 0], np.int32), np.ones((2, 2)))
    assert np.array_equal(got["Y"], np.array([[6, 8], [0, 1]], float))  # exact, as reference


def _random_problem(T, d, k, ranks, counts=None, shuffle=True, seed=0):
    rs = np.random.RandomState(seed)
    S = len(ranks)
    if counts is None:
        counts = rs.multinomial(T - S, [1.0 / S] * S) + 1
    slots = np.repeat(np.arange(S), counts).astype(np.int32)
    if shuffle:
        rs.shuffle(slots)
    X = bf(rs.randn(len(slots), d))
    W = bf(rs.randn(d, k) / np.sqrt(d))
    A = [bf(rs.randn(d, r) / np.sqrt(d)) for r in ranks]
    B = [bf(rs.randn(r, k) / np.sqrt(r)) for r in ranks]
    dY = bf(rs.randn(len(slots), k))
    return X, W, A, B, slots, dY


@pytest.mark.parametrize("shuffle,gathered", [(False, False), (True, False), (True, True)])
def test_c1_full_size(shuffle, gathered):
    wl = config("C1")
    rs = np.random.RandomState(11)
    slots = wl.token_slots(shuffle=shuffle)
    T, d, k = wl.tokens, 1024, 1024
    X = bf(rs.randn(T, d))
    W = bf(rs.randn(d, k) / np.sqrt(d))
    A = [bf(rs.randn(d, r) / np.sqrt(d)) for r in wl.ranks]
    B = [bf(rs.randn(r, k) / np.sqrt(r)) for r in wl.ranks]
    dY = bf(rs.randn(T, k))
    got = gpu_run(X, W, A, B, slots, dY, beta_runs=2 if gathered else 1, gathered=gathered)
    check(got, X, W, A, B, slots, dY, scale_grads=2.0 if gathered else 1.0)


def test_gathered_plan_matches_sorted_batch_bitwise():
    """A gathered plan over an interleaved batch is the job-contiguous plan of the sorted
    batch with a row map on the Y / dX stores: outputs are the sorted run's, bit for bit,
    scattered back to token order; adapter gradients are bitwise equal."""
    rs = np.random.RandomState(7)
    T, d, k, ranks = 1000, 512, 384, [8, 24, 64, 128]
    slots = rs.randint(0, len(ranks), T).astype(np.int32)
    perm = np.argsort(slots, kind="stable")
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev).bfloat16()  # noqa: E731
    X, dY = t(bf(rs.randn(T, d))), t(bf(rs.randn(T, k)))
    W = t(bf(rs.randn(d, k) / np.sqrt(d)))
    A = [t(bf(rs.randn(d, r) / np.sqrt(d))) for r in ranks]
    B = [t(bf(rs.randn(r, k) / np.sqrt(r))) for r in ranks]
    res = []
    for gathered in (False, True):
        lay = FusedLoRALayer(d, k, ranks)
        lay.set_base(W)
        for s in range(len(ranks)):
            lay.set_adapter(s, A[s], B[s])
        if gathered:
            plan = lay.plan(slots, gathered=True)
            assert np.array_equal(plan.row_map(), perm)
            Xg, dYg = torch.empty_like(X), torch.empty_like(dY)
            plan.gather([(X, Xg), (dY, dYg)])
            assert torch.equal(Xg, X[torch.from_numpy(perm).to(dev)])
        else:
            plan = lay.plan(slots[perm])
            idx = torch.from_numpy(perm).to(dev)
            Xg, dYg = X[idx].contiguous(), dY[idx].contiguous()
        Y, H = lay.forward(plan, Xg)
        dX = lay.backward(plan, dYg, Xg, H)
        torch.cuda.synchronize()
        if not gathered:  # scatter the sorted run's outputs to token order
            idx = torch.from_numpy(perm).to(dev)
            Ys, dXs = torch.empty_like(Y), torch.empty_like(dX)
            Ys[idx], dXs[idx] = Y, dX
            Y, dX = Ys, dXs
        res.append((Y, dX, [torch.cat([g.flatten() for g in lay.read_grad(s)])
                            for s in range(len(ranks))]))
        lay.close()
    (Y0, dX0, g0), (Y1, dX1, g1) = res
    assert torch.equal(Y0, Y1) and torch.equal(dX0, dX1)
    assert all(torch.equal(a, b) for a, b in zip(g0, g1))


@pytest.mark.parametrize("cell", [(1024, 2, 2048, 1), (1024, 8, 2048, 2), (1024, 16, 2048, 3),
                                  (1024, 32, 2048, 4), (4096, 4, 2048, 5)])
def test_c5_heterogeneity_cells(cell):
    d, J, T, seed = cell
    wl = c5_cell(d, J, T, seed)
    X, W, A, B, slots, dY = _random_problem(wl.tokens, d, d, wl.ranks,
                                            counts=[j.tokens for j in wl.jobs], seed=seed)
    got = gpu_run(X, W, A, B, slots, dY)
    check(got, X, W, A, B, slots, dY)


@pytest.mark.parametrize("case", [
    dict(T=1, d=8, k=8, ranks=[1]),                    # one token, rank 1
    dict(T=129, d=64, k=40, ranks=[3, 5]),             # ragged tile edge, odd ranks
    dict(T=300, d=256, k=264, ranks=[256, 8, 4]),      # rank = d, N not a tile multiple
    dict(T=1000, d=136, k=72, ranks=[16] * 12),        # many slots, d not a K-block multiple
])
def test_edge_shapes(case):
    X, W, A, B, slots, dY = _random_problem(case["T"], case["d"], case["k"], case["ranks"],
                                            seed=case["T"])
    got = gpu_run(X, W, A, B, slots, dY)
    check(got, X, W, A, B, slots, dY)


def test_slots_absent_from_batch_and_accumulation():
    """Registry slots with no tokens get zero gradients; beta=1 accumulates exactly 2x."""
    X, W, A, B, slots, dY = _random_problem(700, 128, 128, [8, 16, 32, 64], seed=3)
    slots = np.where(slots == 2, 1, slots).astype(np.int32)  # slot 2 absent
    got = gpu_run(X, W, A, B, slots, dY, beta_runs=2)
    check(got, X, W, A, B, slots, dY, scale_grads=2.0)


def _c2_layer(proj="gate", seed=0):
    wl = config("C2")
    name, d, k = [p for p in wl.projections if p[0] == proj][0]
    g = torch.Generator(device="cuda").manual_seed(seed)
    lay = FusedLoRALayer(d, k, wl.ranks)
    lay.set_base((torch.randn(d, k, generator=g, device="cuda") * d ** -0.5).bfloat16())
    As, Bs = [], []
    for s, r in enumerate(wl.ranks):
        A = (torch.randn(d, r, generator=g, device="cuda") * d ** -0.5).bfloat16()
        B = (torch.randn(r, k, generator=g, device="cuda") * r ** -0.5).bfloat16()
        lay.set_adapter(s, A, B)
        As.append(A)
        Bs.append(B)
    X = torch.randn(wl.tokens, d, generator=g, device="cuda").bfloat16()
    dY = torch.randn(wl.tokens, k, generator=g, device="cuda").bfloat16()
    return wl, lay, As, Bs, X, dY


@pytest.mark.parametrize("proj", ["gate", "down"])
def test_c2_full_size_properties(proj):
    """Full C2 size: bit-exact scaling and permutation equivariance, plus an fp32 torch
    restatement of every job's block (cuBLAS fp32 as an independent floating-point check)."""
    wl, lay, As, Bs, X, dY = _c2_layer(proj)
    slots = wl.token_slots()
    plan = lay.plan(slots)
    Y1, H1 = lay.forward(plan, X, y_dtype=torch.float32)
    Y2, _ = lay.forward(plan, X * 2, y_dtype=torch.float32)
    assert torch.equal(Y2, 2 * Y1), "Y(2X) != 2 Y(X) bitwise"
    dX1 = lay.backward(plan, dY, X, H1)
    dA1, dB1 = [t.clone() for t in lay.packed_grads()]
    dX2 = lay.backward(plan, dY * 2, X, H1)
    dA2, dB2 = lay.packed_grads()
    assert torch.equal(dX2.float(), 2 * dX1.float()) and torch.equal(dB2, 2 * dB1) \
        and torch.equal(dA2, 2 * dA1)
    # permutation equivariance (token order is free, fused_lora.hpp:28-31)
    perm = np.random.RandomState(1).permutation(wl.tokens)
    plan_p = lay.plan(slots[perm])
    pt = torch.from_numpy(perm).cuda()
    Yp, _ = lay.forward(plan_p, X[pt].contiguous(), y_dtype=torch.float32)
    assert torch.equal(Yp, Y1[pt]), "Y not permutation-equivariant bitwise"
    # fp32 torch restatement per job (W regenerated from the same seed as _c2_layer)
    Xf = X.float()
    g = torch.Generator(device="cuda").manual_seed(0)
    d, k = X.shape[1], dY.shape[1]
    Wf = (torch.randn(d, k, generator=g, device="cuda") * d ** -0.5).bfloat16().float()
    Yr = Xf @ Wf
    st = torch.from_numpy(slots).cuda()
    for s in range(len(wl.ranks)):
        idx = (st == s).nonzero().flatten()
        h = (Xf[idx] @ As[s].float()).bfloat16().float()
        Yr[idx] += h @ Bs[s].float()
    err = (Y1 - Yr).abs().max().item() / max(1.0, Yr.abs().max().item())
    assert err <= 3e-3, err  # same H near-tie bound as the oracle comparison


def test_fused_adamw_matches_restatement():
    """Two AdamW steps of the fused multi-job optimizer vs a float64 numpy restatement
    (per-job lr / weight decay, bias-corrected moments), then a forward with the refreshed
    bf16 operand layouts vs the oracle on the updated adapters."""
    X, W, A, B, slots, dY = _random_problem(600, 128, 136, [8, 24, 64], seed=9)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    lay = FusedLoRALayer(128, 136, [8, 24, 64])
    lay.set_base(t(W).bfloat16())
    for s in range(3):
        lay.set_adapter(s, t(A[s]).float(), t(B[s]).float())
    lr, wd, b1, b2, eps = [1e-2, 2e-2, 5e-3], [0.0, 0.1, 0.01], 0.9, 0.99, 1e-8
    lay.set_optimizer(lr, wd, b1, b2, eps)
    plan = lay.plan(slots)
    Xd, dYd = t(X).bfloat16(), t(dY).bfloat16()
    P = {s: [A[s].astype(np.float32).astype(np.float64), B[s].astype(np.float32).astype(np.float64)]
         for s in range(3)}
    M = {s: [np.zeros_like(P[s][0]), np.zeros_like(P[s][1])] for s in range(3)}
    V = {s: [np.zeros_like(P[s][0]), np.zeros_like(P[s][1])] for s in range(3)}
    scale = 0.5
    for step in (1, 2):
        Y, H = lay.forward(plan, Xd)
        lay.backward(plan, dYd, Xd, H)
        torch.cuda.synchronize()
        grads = {s: [g.double().cpu().numpy() for g in lay.read_grad(s)] for s in range(3)}
        lay.optimizer_step(grad_scale=scale)
        torch.cuda.synchronize()
        for s in range(3):
            for i in range(2):
                g = grads[s][i] * scale
                M[s][i] = b1 * M[s][i] + (1 - b1) * g
                V[s][i] = b2 * V[s][i] + (1 - b2) * g * g
                mh, vh = M[s][i] / (1 - b1 ** step), V[s][i] / (1 - b2 ** step)
                P[s][i] = P[s][i] - lr[s] * (mh / (np.sqrt(vh) + eps) + wd[s] * P[s][i])
            got = [x.double().cpu().numpy() for x in lay.read_adapter(s)]
            for i in range(2):
                err = np.abs(got[i] - P[s][i]).max() / max(1e-6, np.abs(P[s][i]).max())
                assert err < 1e-5, (step, s, i, err)
    # the kernels now read the refreshed bf16 copies of the updated adapters
    Y, _ = lay.forward(plan, Xd, y_dtype=torch.float32)
    Ab = [bf(lay.read_adapter(s)[0].double().cpu().numpy()) for s in range(3)]
    Bb = [bf(lay.read_adapter(s)[1].double().cpu().numpy()) for s in range(3)]
    Ye = O.fused_forward(X, W, Ab, Bb, slots, round_bf16=True)
    assert maxrel(Y.double().cpu().numpy(), Ye) <= 3e-3
    lay.close()


def test_overlapped_schedule_is_bit_identical():
    """The two-stream schedule (low-rank launches on a side stream with a capped SM
    budget) runs the same tiles in the same order per tile: results are bitwise equal."""
    from paper_2602_07263_b200 import capi
    from paper_2602_07263_b200.runner import LayerSetStep
    from paper_2602_07263_b200.workload import Job, Workload

    wl = Workload("mini", [("q", 512, 768), ("k", 512, 256), ("o", 768, 512)],
                  [Job("a", 8, 2, 256), Job("b", 64, 3, 256), Job("c", 16, 1, 256)], layers=2)
    out = []
    for overlap in (False, True):
        st = LayerSetStep(wl, device=0, seed=5, chain=False)
        main = torch.cuda.current_stream()
        if overlap:
            st.enable_overlap(16)
            st.forward_overlapped(main)
            st.backward_overlapped(main)
        else:
            st.forward(main)
            st.backward(main)
        torch.cuda.synchronize()
        out.append({"Y": {k: v.clone() for k, v in st.Y.items()},
                    "dX": {k: v.clone() for k, v in st.dX.items()},
                    "g": {k: [t.clone() for t in lay.packed_grads()] for k, lay in st.layers.items()}})
        capi.call("tlora_set_sm_budget", 0, 0, 0)
    a, b = out
    for k in a["Y"]:
        assert torch.equal(a["Y"][k], b["Y"][k]) and torch.equal(a["dX"][k], b["dX"][k]), k
    for k in a["g"]:
        assert all(torch.equal(x, y) for x, y in zip(a["g"][k], b["g"][k])), k


def test_cuda_graph_replay_matches_eager():
    """A captured training step (fwd + bwd + AdamW, device-side optimizer counters)
    replays bit-identically to the same steps run eagerly."""
    from paper_2602_07263_b200.runner import LayerSetStep
    from paper_2602_07263_b200.workload import Job, Workload

    wl = Workload("mini", [("q", 512, 768), ("o", 768, 512)],
                  [Job("a", 8, 2, 256), Job("b", 64, 3, 256)])
    res = []
    for use_graph in (False, True):
        st = LayerSetStep(wl, device=0, seed=3)
        st.enable_optimizer(1e-3, 0.01)
        if use_graph:
            g = st.capture(warmup=1)  # eager step 1, then the captured step
            for _ in range(2):
                g.replay()
        else:
            for _ in range(3):
                st.step()
        torch.cuda.synchronize()
        res.append({k: [t.clone() for t in (lay.read_adapter(0) + lay.read_adapter(1))]
                    for k, lay in st.layers.items()})
    for k in res[0]:
        assert all(torch.equal(x, y) for x, y in zip(res[0][k], res[1][k])), k


@pytest.mark.parametrize("tokens", [(256, 256, 256), (300, 77, 513)])
def test_chained_lowrank_tiles_are_bit_identical(tokens, monkeypatch):
    """Chained schedule (next projection's shrink / dH as extra CTA-pair tiles of the fused
    GEMM launch: tlora_forward_gemm_shrink / tlora_backward_dx_dh) vs one launch per op:
    Y, dX, H stashes and adapter gradients bitwise equal, ragged token counts included.
    The side-stream variant runs with dH ring depths 2 (a wait before every dX launch) and
    8 (no waits over these 6 projections)."""
    from paper_2602_07263_b200.runner import LayerSetStep
    from paper_2602_07263_b200.workload import Job, Workload

    wl = Workload("mini", [("q", 512, 768), ("k", 512, 256), ("o", 768, 512)],
                  [Job("a", 8, 2, tokens[0]), Job("b", 200, 3, tokens[1]),
                   Job("c", 16, 1, tokens[2])], layers=2)
    out = []
    for chain, side, ring in ((False, False, 0), (True, False, 0), (True, True, 2), (True, True, 8)):
        st = LayerSetStep(wl, device=0, seed=7, chain=chain)
        if side:  # dB+dA launches on a side stream (runner.enable_side_grads)
            monkeypatch.setenv("TLORA_DH_RING", str(ring))
            st.enable_side_grads()
            assert st.dh_ring == ring
        st.forward()
        st.backward()
        torch.cuda.synchronize()
        out.append({"Y": {k: v.clone() for k, v in st.Y.items()},
                    "dX": {k: v.clone() for k, v in st.dX.items()},
                    "H": {k: v.clone() for k, v in st.H.items()},
                    "g": {k: [t.clone() for t in lay.packed_grads()] for k, lay in st.layers.items()}})
    a = out[0]
    for b in out[1:]:
        for k in a["Y"]:
            assert torch.equal(a["Y"][k], b["Y"][k]) and torch.equal(a["dX"][k], b["dX"][k]), k
        for k in a["H"]:
            assert torch.equal(a["H"][k], b["H"][k]), k
        for k in a["g"]:
            assert all(torch.equal(x, y) for x, y in zip(a["g"][k], b["g"][k])), k


def test_gemm_shrink_zero_next_clears_garbage():
    """tlora_forward_gemm_shrink / tlora_backward_dx_dh with zero_next=1 on a garbage-filled
    output equal the standalone shrink / dH (which memset) bitwise, and the fused GEMM part
    equals tlora_forward_gemm / tlora_backward_dx."""
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(11)
    ranks = [8, 64, 24, 128]
    d0, k0, d1, k1 = 640, 384, 384, 1152
    lays = []
    for d, k in ((d0, k0), (d1, k1)):
        lay = FusedLoRALayer(d, k, ranks)
        lay.set_base((torch.randn(d, k, generator=g, device=dev) * d ** -0.5).bfloat16())
        for s_, r in enumerate(ranks):
            lay.set_adapter(s_, (torch.randn(d, r, generator=g, device=dev) * 0.05).bfloat16(),
                            (torch.randn(r, k, generator=g, device=dev) * 0.05).bfloat16())
        lays.append(lay)
    slots = np.random.default_rng(3).integers(0, 4, 700).astype(np.int32)
    T = len(slots)
    p0, p1 = lays[0].plan(slots), lays[1].plan(np.sort(slots))
    R = lays[0].R
    X0 = torch.randn(T, d0, generator=g, device=dev).bfloat16()
    X1 = torch.randn(T, d1, generator=g, device=dev).bfloat16()
    H0 = torch.empty(T, R, dtype=torch.bfloat16, device=dev)
    lays[0].shrink(p0, X0, H0)
    Ya, Yb = (torch.empty(T, k0, dtype=torch.bfloat16, device=dev) for _ in range(2))
    Ha = torch.empty(T, R, dtype=torch.bfloat16, device=dev)
    Hb = torch.full((T, R), 7.0, dtype=torch.bfloat16, device=dev)
    lays[0].fused_gemm(p0, X0, H0, Ya)
    lays[1].shrink(p1, X1, Ha)
    lays[0].fused_gemm_shrink(p0, X0, H0, Yb, lays[1], p1, X1, Hb, zero_next=True)
    torch.cuda.synchronize()
    assert torch.equal(Ya, Yb) and torch.equal(Ha, Hb)
    dY0 = torch.randn(T, k0, generator=g, device=dev).bfloat16()
    dY1 = torch.randn(T, k1, generator=g, device=dev).bfloat16()
    dH0 = torch.empty(T, R, dtype=torch.bfloat16, device=dev)
    lays[0].dh(p0, dY0, dH0)
    dXa, dXb = (torch.empty(T, d0, dtype=torch.bfloat16, device=dev) for _ in range(2))
    dHa = torch.empty(T, R, dtype=torch.bfloat16, device=dev)
    dHb = torch.full((T, R), -3.0, dtype=torch.bfloat16, device=dev)
    lays[0].dx(p0, dY0, dH0, dXa)
    lays[1].dh(p1, dY1, dHa)
    lays[0].dx_dh(p0, dY0, dH0, dXb, lays[1], p1, dY1, dHb, zero_next=True)
    torch.cuda.synchronize()
    assert torch.equal(dXa, dXb) and torch.equal(dHa, dHb)
    for lay in lays:
        lay.close()


def test_uploaded_plan_is_bit_identical_to_plan_oracle():
    """What the kernels actually read: every tile table and the token-slot array copied
    back from device memory (tlora_plan_read_device) memcmp-equal to the plan oracle
    (bit-exact plan + owner-id readback)."""
    rs = np.random.RandomState(4)
    c2 = config("C2")
    cases = [(1024, 1024, [8, 16, 32, 64], rs.randint(0, 4, 7680).astype(np.int32)),
             (4096, 4096, c2.ranks, c2.token_slots()),
             (256, 264, [4, 256, 8, 1], np.array([1] * 300 + [3] * 5, np.int32))]
    dev = torch.device("cuda", 0)
    for d, k, ranks, slots in cases:
        lay = FusedLoRALayer(d, k, ranks)
        lay.set_base(torch.zeros(d, k, dtype=torch.bfloat16, device=dev))
        for s_, r in enumerate(ranks):
            lay.set_adapter(s_, torch.zeros(d, r, dtype=torch.bfloat16, device=dev),
                            torch.zeros(r, k, dtype=torch.bfloat16, device=dev))
        plan = lay.plan(slots)
        for launch in range(8):
            tiles, dev_slots = plan.device_tiles(launch)
            want = O.plan_tiles(len(slots), d, k, ranks, slots, launch)
            assert tiles.shape == want.shape and np.array_equal(tiles, want), (d, k, launch)
            assert np.array_equal(dev_slots, slots)
        lay.close()


@pytest.mark.parametrize("shape", [("C3", "gate"), ("C3", "down"), ("C4", "q"), ("C4", "down"),
                                   ("C2", "k")])
def test_model_projection_shapes(shape):
    """The real projection shapes of the Llama-3-8B (C3) and Qwen3-32B (C4) stacks and
    Qwen3-8B's narrow k projection, with each config's 16 / 8 heterogeneous jobs on a
    small ragged token batch (10-30 tokens per job, not tile multiples), vs the oracle."""
    name, proj = shape
    wl = config(name)
    _, d, k = [p for p in wl.projections if p[0] == proj][0]
    rs = np.random.RandomState(len(proj) + d)
    counts = [int(rs.randint(10, 30)) for _ in wl.jobs]
    X, W, A, B, slots, dY = _random_problem(sum(counts), d, k, wl.ranks, counts=counts,
                                            seed=d + k)
    got = gpu_run(X, W, A, B, slots, dY)
    check(got, X, W, A, B, slots, dY)


_LPT_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2602_07263_b200.layer import FusedLoRALayer
rs = np.random.RandomState(3)
T, d, k, ranks = 8192, 4096, 2048, [8, 24, 64, 128, 16]
slots = np.sort(rs.randint(0, len(ranks), T)).astype(np.int32)
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(a.astype(np.float32)).to(dev).bfloat16()
lay = FusedLoRALayer(d, k, ranks)
lay.set_base(t(rs.randn(d, k) / np.sqrt(d)))
for s, r in enumerate(ranks):
    lay.set_adapter(s, t(rs.randn(d, r) / np.sqrt(d)), t(rs.randn(r, k) / np.sqrt(r)))
plan = lay.plan(slots)
X, dY = t(rs.randn(T, d)), t(rs.randn(T, k))
Y, H = lay.forward(plan, X)
dX = lay.backward(plan, dY, X, H)
torch.cuda.synchronize()
np.save(sys.argv[2], np.concatenate([t.float().cpu().numpy().ravel()
                                     for t in [Y, dX] + list(lay.packed_grads())]))
"""


@pytest.mark.parametrize("knob", [("TLORA_GRAD_LPT", "1", "0"), ("TLORA_DYN_SCHED", "1", "0")])
def test_schedules_are_bitwise_identical(tmp_path, knob):
    """Tile schedules only change which CTA runs a tile and when; every output element is
    still produced by one tile with the same accumulation order. LPT-balanced gradient tile
    lists (tlora::grad_schedule) vs round-robin, and the fused GEMM's dynamic ticket
    scheduler vs its static round-robin: Y, dX and the gradients are equal bit for bit."""
    import os
    import subprocess
    var, a, b = knob
    script = tmp_path / "sched.py"
    script.write_text(_LPT_SCRIPT)
    out = {}
    for val in (a, b):
        f = tmp_path / f"g{val}.npy"
        env = dict(os.environ, **{var: val})
        subprocess.run([sys.executable, str(script), str(ROOT), str(f)], check=True, env=env,
                       timeout=300)
        out[val] = np.load(f)
    assert out[a].size > 0 and np.array_equal(out[a], out[b])
