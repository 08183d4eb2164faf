"""Full-size parity of the EXACT training step bench.py times (VERDICT r1 "next" item 1).

The step under test is built the way bench.py builds it: `LayerSetStep(chain=True)`,
fused multi-job AdamW, side-stream dB+dA with the dH ring (default depth 8), the
chained schedule (next projection's shrink / dH as extra tiles of the fused GEMM, first
dH prefetched by the last forward launch), captured once into a CUDA graph and REPLAYED.
The replayed step is compared with an independent fp32 torch restatement of
fused_lora.hpp:84-119 (+ its backward) on the same bf16 inputs, at the benched sizes:

  * C2 (Qwen3-8B, 7 projections, T = 16384, T_j up to 4096 -> split-K gradient planes),
  * two layers of C3 (Llama-3-8B, 14 (layer, projection) pairs, T = 61440),
  * C4 up + down projections (Qwen3-32B, 25600-wide, T = 61440, T_j up to 8192).

Reference numerics (SURVEY.md §8(c) tolerances, stated here):
  Y, dX   max-abs <= 1e-2 * max(1, max|ref|)  and  ||diff||_F <= 4e-3 * ||ref||_F
  dA, dB  max-abs <= 2e-2 * max(1, max|ref|)  and  ||diff||_F <= 8e-3 * ||ref||_F
  H (the stash the backward consumed) ||diff||_F <= 4e-3 * ||ref||_F, zero outside the
          token's own packed-rank columns.
The restatement rounds H = X_j·A_j and dH = dY_j·B_jᵀ to bf16 exactly where the device
stashes them, and runs every product in fp32 (TF32 off).
Post-AdamW fp32 adapters: vs a float64 AdamW restatement applied to the device's own
gradients (<= 1e-5 relative), and vs the same restatement on the REFERENCE gradients
(first Adam step: |update| <= lr·(1 + wd·|p|), so the only admissible difference is a
sign flip of near-zero gradient elements: elementwise <= 2·lr + wd·lr·|p|, and on < 1% of
the elements).
The profiled graph (CUDA-event nodes around every launch, replayed as the bench's last
timed step) is replayed from the same restored state and must be bitwise identical.
"""
import numpy as np
import pytest
import torch

from paper_2602_07263_b200.runner import LayerSetStep
from paper_2602_07263_b200.workload import INPUT_GROUP, Workload, config

pytestmark = pytest.mark.gpu

TOL = {"Y": (1e-2, 4e-3), "dX": (1e-2, 4e-3), "dA": (2e-2, 8e-3), "dB": (2e-2, 8e-3)}


def _errs(got, ref):
    got, ref = got.float(), ref.float()
    diff = got - ref
    mx = (diff.abs().max() / max(1.0, ref.abs().max().item())).item()
    n = ref.norm().item()
    fr = (diff.norm() / (n if n > 0 else 1.0)).item()
    return mx, fr


def _check(what, got, ref, key, report):
    mx, fr = _errs(got, ref)
    report.append((key, what, mx, fr))
    tmx, tfr = TOL[what]
    assert mx <= tmx and fr <= tfr, (key, what, mx, fr)


def _job_ranges(wl):
    out, t = [], 0
    for j in wl.jobs:
        out.append((t, t + j.tokens))
        t += j.tokens
    return out


def _snapshot(st):
    """fp32 master adapters of every (layer, projection), slot order."""
    return {key: [tuple(t.clone() for t in lay.read_adapter(s)) for s in range(len(lay.ranks))]
            for key, lay in st.layers.items()}


def _restore(st, snap, lrs, wd):
    for key, lay in st.layers.items():
        for s, (A, B) in enumerate(snap[key]):
            lay.set_adapter(s, A, B)
        lay.set_optimizer(lrs, wd)  # zero moments and step counters


def _outputs(st, keys):
    torch.cuda.synchronize()
    return {
        "Y": {n: t.clone() for n, t in st.Y.items()},
        "dX": {n: t.clone() for n, t in st.dX.items()},
        "H": {k: st.H[k].clone() for k in keys},
        "g": {k: [tuple(t.clone() for t in st.layers[k].read_grad(s))
                  for s in range(len(st.layers[k].ranks))] for k in keys},
        "P": _snapshot(st),
    }


def _segments_python(wl):
    """Job-contiguous layout of LayerSetStep: one row range per slot."""
    return [[r] for r in _job_ranges(wl)]


def _segments_executor(st, n):
    """Row ranges of every slot in the executor's nano-major layout for nano count n."""
    n_used, t0, ns, _ = st.layout(n)
    segs = [[] for _ in st.wl.jobs]
    for i in range(n_used):
        row = int(t0[i])
        for s, j in enumerate(st.wl.jobs):
            rows = int(ns[i, s]) * j.seq_len
            if rows:
                segs[s].append((row, row + rows))
            row += rows
    return n_used, segs


def _build(wl, seed, driver, nano):
    """The step exactly as bench.py builds it: returns (step, run_plain, run_profiled,
    segments). run_plain replays the captured graph; run_profiled is the bench's last timed
    step (Python driver: the second capture with CUDA-event nodes; executor: the eager,
    event-bracketed run)."""
    from paper_2602_07263_b200 import capi
    if driver == "python":
        st = LayerSetStep(wl, device=0, seed=seed, chain=True, keep_weights=True)
        st.enable_optimizer(1e-4, 0.01)  # bench.py: step.enable_optimizer() (same defaults)
        st.enable_side_grads()           # bench.py default (TLORA_SIDE_GRADS=1), dH ring 8
        assert st.dh_ring == 8
        graph = st.capture(warmup=1, profile=False)
        graph_prof = st.capture(warmup=0, profile=True)
        return st, graph.replay, graph_prof.replay, _segments_python(wl)
    from paper_2602_07263_b200.step import TrainingStep
    st = TrainingStep(wl, device=0, nano_fixed=nano, graphs=True, dh_ring=8)
    st.init_random(seed, keep_weights=True)
    st.enable_optimizer(1e-4, 0.01)
    first = st.run()        # eager (allocates plan scratch), then captured for this N
    assert not first.replayed_graph and first.nano_used == min(nano, sum(j.batch for j in wl.jobs))

    def plain():
        assert st.run().replayed_graph

    def profiled():
        capi.call("tlora_profile_begin")
        assert not st.run(eager=True).replayed_graph
    n_used, segs = _segments_executor(st, nano)
    return st, plain, profiled, segs


def _x(st, name):
    return st.x_of(name) if hasattr(st, "x_of") else st.X[0][INPUT_GROUP.get(name, name)]


def _dy(st, name):
    return st.dy_of(name) if hasattr(st, "dy_of") else st.dY[0][name]


def _run_case(wl, seed=11, driver="python", nano=1):
    torch.backends.cuda.matmul.allow_tf32 = False
    from paper_2602_07263_b200 import capi
    st, run_plain, run_prof, segs = _build(wl, seed, driver, nano)
    lrs = [1e-4 * (1.0 + 0.25 * (s % 4)) for s in range(len(wl.jobs))]
    wd = 0.01
    keys = st.keys
    # state at the start of the replayed step: adapters after one eager step, AdamW moments
    # and step counters reset (so the replay is a first Adam step, restatable exactly)
    snap = _snapshot(st)
    _restore(st, snap, lrs, wd)
    run_plain()
    got = _outputs(st, keys)
    # the profiled variant replayed from the same state: bitwise identical
    _restore(st, snap, lrs, wd)
    run_prof()
    got2 = _outputs(st, keys)
    capi.call("tlora_profile_end", None, None, None)
    for part in ("Y", "dX"):
        for n in got[part]:
            assert torch.equal(got[part][n], got2[part][n]), (part, n)
    for k in keys:
        assert torch.equal(got["H"][k], got2["H"][k]), k
        for a, b in zip(got["g"][k] + got["P"][k], got2["g"][k] + got2["P"][k]):
            assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]), k

    last_layer, report = wl.layers - 1, []
    for key in keys:
        L, name = key
        lay = st.layers[key]
        W, _ = st.weights[key]
        Wf = W.float()
        X, dY = _x(st, name).float(), _dy(st, name).float()
        P0 = snap[key]
        # bf16 operands the kernels read = round(fp32 master)
        As = [P0[s][0].bfloat16().float() for s in range(len(segs))]
        Bs = [P0[s][1].bfloat16().float() for s in range(len(segs))]
        Yr = X @ Wf if L == last_layer else None      # Y buffers hold the last layer's Y
        dXr = dY @ Wf.t() if L == 0 else None         # dX buffers hold layer 0's dX
        Hg = got["H"][key]
        mask = torch.ones_like(Hg, dtype=torch.bool)
        for s, ranges in enumerate(segs):
            A, B = As[s], Bs[s]
            off, r = lay.offsets[s], lay.ranks[s]
            dAr = torch.zeros(A.shape, device=A.device)
            dBr = torch.zeros(B.shape, device=B.device)
            for t0, t1 in ranges:  # the job's rows (one range, or one per nano-batch)
                h = (X[t0:t1] @ A).bfloat16().float()
                dh = (dY[t0:t1] @ B.t()).bfloat16().float()
                if Yr is not None:
                    Yr[t0:t1] += h @ B
                if dXr is not None:
                    dXr[t0:t1] += dh @ A.t()
                mask[t0:t1, off:off + r] = False
                mx, fr = _errs(Hg[t0:t1, off:off + r], h)
                report.append((key, f"H{s}", mx, fr))
                assert fr <= 4e-3, (key, s, "H", fr)
                dAr += X[t0:t1].t() @ dh
                dBr += h.t() @ dY[t0:t1]
            gA, gB = got["g"][key][s]
            _check("dA", gA, dAr, (key, s), report)
            _check("dB", gB, dBr, (key, s), report)
            # AdamW (first step from zero moments, bias-corrected) in float64
            lr = lrs[s]
            P1 = got["P"][key][s]
            for i, (p0, g_dev, g_ref) in enumerate(((P0[s][0], gA, dAr), (P0[s][1], gB, dBr))):
                p0d = p0.double()

                def adam(g):
                    g = g.double()
                    m, v = 0.1 * g, 0.001 * g * g
                    return p0d - lr * ((m / 0.1) / (torch.sqrt(v / 0.001) + 1e-8) + wd * p0d)

                e_dev = ((P1[i].double() - adam(g_dev)).abs().max() / p0d.abs().max()).item()
                assert e_dev < 1e-5, (key, s, i, e_dev)
                d_ref = (P1[i].double() - adam(g_ref)).abs()
                bound = 2.0 * lr * 1.0001 + wd * lr * p0d.abs() + 1e-7
                assert bool((d_ref <= bound).all()), (key, s, i, d_ref.max().item())
                flips = (d_ref > 0.5 * lr).double().mean().item()
                report.append((key, f"adam_flip{s}{'AB'[i]}", flips, 0.0))
                assert flips < 1e-2, (key, s, i, flips)
        assert not bool(Hg[mask].any()), (key, "H not masked to own columns")
        if Yr is not None:
            _check("Y", got["Y"][name], Yr, key, report)
        if dXr is not None:
            _check("dX", got["dX"][name], dXr, key, report)
        del Yr, dXr, X, dY, Wf
    worst = {}
    for key, what, mx, fr in report:
        w = what.rstrip("0123456789") if not what.startswith("adam") else "adam_flip"
        worst[w] = max(worst.get(w, (0, 0)), (mx, fr))
    print(f"{wl.name} [{driver}, N={nano}]: worst (max-abs rel, frob rel) per quantity: {worst}")
    return st


def test_c2_benched_step_full_size():
    wl = config("C2")
    st = _run_case(wl)
    splits = {name: pl.info().splits_db for name, pl in st.plans.items()}
    assert max(splits.values()) > 1, splits  # split-K dB planes (T_j = 4096) exercised


def test_c3_two_layers_benched_step():
    wl = config("C3")
    wl.layers = 2
    _run_case(wl)


def test_c4_projections_t61440_benched_step():
    full = config("C4")
    wl = Workload("C4[up,down]", [p for p in full.projections if p[0] in ("up", "down")],
                  full.jobs, layers=1, seed=full.seed)
    assert wl.tokens == 61440
    _run_case(wl)


# ---- the C++ step executor (tlora_step_*, the bench's default path) at full size
@pytest.mark.parametrize("nano", [1, 3])
def test_c2_executor_step_full_size(nano):
    """C2 through the C++ executor: N = 1 (the graph the bench replays) and N = 3 rank-aware
    nano-batches (gradients accumulated over three nano-batches of the nano-major layout)."""
    _run_case(config("C2"), driver="cpp", nano=nano)


def test_c3_two_layers_executor_nano4():
    wl = config("C3")
    wl.layers = 2
    _run_case(wl, driver="cpp", nano=4)
