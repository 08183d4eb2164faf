"""The C++ step executor (tlora_step_*) on the GPU: bitwise agreement with the Python
per-launch driver it replaces, the AIMD controller driven by its own measured step times
(nano_pipeline.hpp:99-112, clamped as sim_engine.hpp:314), the rank-aware token layout
as uploaded, the masked optimizer for jobs absent from a step, and the pure-C++ host
(tests/cpp/step_main) matching the Python-driven executor bit for bit."""
import math
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as O  # noqa: E402

from paper_2602_07263_b200.runner import LayerSetStep  # noqa: E402
from paper_2602_07263_b200.step import TrainingStep, sample_weights  # noqa: E402
from paper_2602_07263_b200.workload import INPUT_GROUP, Job, Workload, config  # noqa: E402

pytestmark = pytest.mark.gpu

MINI = Workload("mini", [("q", 512, 768), ("k", 512, 256), ("o", 768, 512), ("down", 640, 768)],
                [Job("a", 8, 2, 256), Job("b", 200, 3, 320), Job("c", 16, 1, 192),
                 Job("d", 64, 2, 128)], layers=2, seed=77)


def _state(st):
    torch.cuda.synchronize()
    return {
        "Y": {n: t.clone() for n, t in st.Y.items()},
        "dX": {n: t.clone() for n, t in st.dX.items()},
        "H": {k: st.H[k].clone() for k in st.keys},
        "g": {k: [t.clone() for s in range(len(st.layers[k].ranks))
                  for t in st.layers[k].read_grad(s)] for k in st.keys},
        "P": {k: [t.clone() for s in range(len(st.layers[k].ranks))
                  for t in st.layers[k].read_adapter(s)] for k in st.keys},
    }


def _equal(a, b):
    for part in ("Y", "dX", "H"):
        for key in a[part]:
            assert torch.equal(a[part][key], b[part][key]), (part, key)
    for part in ("g", "P"):
        for key in a[part]:
            assert all(torch.equal(x, y) for x, y in zip(a[part][key], b[part][key])), (part, key)


@pytest.mark.parametrize("wl", [MINI, config("C2")], ids=["mini", "C2"])
def test_executor_matches_python_driver_bitwise(wl):
    """N = 1: the executor's chained schedule is the Python driver's chained + side-stream
    schedule (same launches, same tiles): every output, stash, gradient and updated adapter
    is bitwise equal, for the eager first step and for graph replays."""
    py = LayerSetStep(wl, device=0, seed=wl.seed, chain=True)
    py.enable_optimizer()
    py.enable_side_grads()
    ex = TrainingStep(wl, device=0, nano_fixed=1, graphs=True)
    ex.init_random(wl.seed)
    ex.enable_optimizer()
    for i in range(3):
        py.step()
        s = ex.run()
        assert s.replayed_graph == (i > 0) and s.nano_used == 1
        _equal(_state(py), _state(ex))


def test_executor_aimd_follows_reference_rule():
    """N comes from the reference controller fed with the executor's own CUDA-event step
    times: restating aimd_step (oracle) on the reported times reproduces every N, clamped to
    the combined batch; the first observation only seeds t_prev."""
    wl = MINI
    ex = TrainingStep(wl, device=0, nano_fixed=0, nano_init=4, graphs=True)
    ex.init_random(wl.seed)
    ex.enable_optimizer()
    total = sum(j.batch for j in wl.jobs)
    n, t_prev = 4, None
    for _ in range(10):
        assert ex.next_n() == n
        s = ex.run()
        assert s.nano_used == min(n, total)
        n, t_prev = O.aimd_step(n, t_prev, s.ms / 1e3)
        n = min(n, total)
        assert s.next_nano == n
    assert len({u for u, _ in ex.trajectory}) >= 2  # the controller moved N


def test_executor_layout_is_the_rank_aware_map():
    """The layout the executor plans with == the oracle's nano map (bit-exact counts) laid
    out nano-major, job-contiguous inside a nano-batch; sample rows tile [0, T)."""
    wl = config("C2")
    ex = TrainingStep(wl, device=0, nano_fixed=1, graphs=False)
    ex.init_random(wl.seed)  # plans need loaded adapters
    batch, weight = [j.batch for j in wl.jobs], sample_weights(wl)
    for n in (1, 2, 3, 5, 17, 40):
        k, t0, ns, sample_row = ex.layout(n)
        ko, per, sample_nano, nso = O.nano_assign(batch, weight, n)
        assert k == ko and np.array_equal(ns, nso)
        sizes = np.array([ns[i] @ np.array([j.seq_len for j in wl.jobs]) for i in range(k)])
        assert np.array_equal(np.diff(t0), sizes) and t0[-1] == wl.tokens
        seqs = np.repeat([j.seq_len for j in wl.jobs], batch)
        order = np.argsort(sample_row)
        assert np.array_equal(np.cumsum(seqs[order])[:-1], sample_row[order][1:])
        for q in range(len(sample_row)):  # sample q lies inside its nano-batch's row range
            i = sample_nano[q]
            assert t0[i] <= sample_row[q] < t0[i + 1]


def test_masked_optimizer_skips_absent_jobs():
    """A job with no tokens in the step takes no AdamW step (masters and step counter
    unchanged); when it reappears its first update uses bias correction t = 1."""
    from paper_2602_07263_b200.layer import FusedLoRALayer
    rs = np.random.RandomState(3)
    d, k, ranks = 128, 136, [8, 24, 16]
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    lay = FusedLoRALayer(d, k, ranks)
    lay.set_base(t(rs.randn(d, k) / np.sqrt(d)).bfloat16())
    for s, r in enumerate(ranks):
        lay.set_adapter(s, t(rs.randn(d, r) / np.sqrt(d)).float(), t(rs.randn(r, k) / np.sqrt(r)).float())
    lr, wd = [1e-2, 2e-2, 5e-3], [0.0, 0.1, 0.01]
    lay.set_optimizer(lr, wd, 0.9, 0.99, 1e-8)
    X = t(rs.randn(400, d)).bfloat16()
    dY = t(rs.randn(400, k)).bfloat16()
    slots_a = np.repeat([0, 2], [250, 150]).astype(np.int32)    # job 1 absent
    slots_b = np.repeat([0, 1, 2], [100, 200, 100]).astype(np.int32)
    before = [[x.double() for x in lay.read_adapter(s)] for s in range(3)]
    plan = lay.plan(slots_a)
    Y, H = lay.forward(plan, X)
    lay.backward(plan, dY, X, H)
    lay.optimizer_step(plan=plan)
    torch.cuda.synchronize()
    mid = [[x.double() for x in lay.read_adapter(s)] for s in range(3)]
    assert all(torch.equal(a, b) for a, b in zip(before[1], mid[1]))       # untouched
    assert not torch.equal(before[0][0], mid[0][0])                         # stepped
    plan_b = lay.plan(slots_b)
    Y, H = lay.forward(plan_b, X)
    lay.backward(plan_b, dY, X, H)
    g1 = [x.double() for x in lay.read_grad(1)]
    lay.optimizer_step(plan=plan_b)
    torch.cuda.synchronize()
    after = [x.double() for x in lay.read_adapter(1)]
    for p0, g, p1 in zip(mid[1], g1, after):  # first step for job 1: t = 1, zero moments
        m, v = 0.1 * g, 0.01 * g * g
        ref = p0 - lr[1] * ((m / 0.1) / (torch.sqrt(v / 0.01) + 1e-8) + wd[1] * p0)
        assert ((p1 - ref).abs().max() / p0.abs().max()).item() < 1e-5


def test_cpp_host_step_matches_python_driven_executor(tmp_path):
    """tests/cpp/step_main drives the executor purely from C++ (weights and inputs from
    tlora_fill_normal, no Python, no torch) and dumps Y / dX / gradients / adapters after
    two steps at N = 2; the same executor driven from Python with the same fills gives the
    same bytes."""
    binp = ROOT / "tests" / "cpp" / "_build" / "step_main"
    if not binp.exists():
        subprocess.run(["make", "-C", str(ROOT), "tests/cpp/_build/step_main"], check=True)
    out = tmp_path / "cpp.bin"
    p = subprocess.run([str(binp), "dump", str(out)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    cpp = np.fromfile(out, dtype=np.uint8)
    from paper_2602_07263_b200 import capi
    import ctypes as C
    wl = Workload("cpp-mini", [("q", 512, 768), ("k", 512, 256), ("o", 768, 512)],
                  [Job("a", 8, 2, 256), Job("b", 200, 3, 320), Job("c", 16, 1, 192)],
                  layers=2, seed=5)
    ex = TrainingStep(wl, device=0, nano_fixed=2, graphs=True)
    fill = capi.lib().tlora_fill_normal
    seed = 1000
    for key in ex.keys:  # the C++ program's fill order (tests/cpp/step_main.cpp)
        lay = ex.layers[key]
        W = torch.empty(lay.d, lay.k, dtype=torch.bfloat16, device="cuda")
        fill(C.c_void_p(W.data_ptr()), capi.BF16, W.numel(), seed, C.c_float(1.0 / math.sqrt(lay.d)), None)
        seed += 1
        lay.set_base(W)
        for s, r in enumerate(lay.ranks):
            A = torch.empty(lay.d, r, dtype=torch.float32, device="cuda")
            B = torch.empty(r, lay.k, dtype=torch.float32, device="cuda")
            fill(C.c_void_p(A.data_ptr()), capi.F32, A.numel(), seed, C.c_float(1.0 / math.sqrt(lay.d)), None)
            fill(C.c_void_p(B.data_ptr()), capi.F32, B.numel(), seed + 1, C.c_float(1.0 / math.sqrt(r)), None)
            seed += 2
            lay.set_adapter(s, A, B)
    for g in ex.groups:
        x = ex.X[0][g]
        fill(C.c_void_p(x.data_ptr()), capi.BF16, x.numel(), seed, C.c_float(1.0), None)
        seed += 1
    for n in ex.names:
        y = ex.dY[0][n]
        fill(C.c_void_p(y.data_ptr()), capi.BF16, y.numel(), seed, C.c_float(1.0), None)
        seed += 1
    ex.enable_optimizer(1e-3, 0.01)
    ex.run()
    ex.run()
    st = _state(ex)
    parts = [st["Y"][n] for n in ex.names] + [st["dX"][n] for n in ex.names]
    for key in ex.keys:
        parts += st["g"][key] + st["P"][key]
    chunks = [t.contiguous().view(torch.uint8).cpu().numpy().ravel() for t in parts]
    py = np.concatenate(chunks)
    assert py.size == cpp.size
    off, bad = 0, []
    for i, c in enumerate(chunks):  # name the first differing parts (diagnostics)
        if not np.array_equal(c, cpp[off:off + c.size]):
            bad.append(i)
        off += c.size
    assert not bad, f"differing parts (Y x{len(ex.names)}, dX x{len(ex.names)}, then grads/adapters per key): {bad[:10]}"


def test_executor_data_parallel_multi_gpu():
    """tests/step_dp_check.py under torchrun on every visible GPU (>= 2)."""
    import socket
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (run via gpurun --gpus 2)")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    n = min(torch.cuda.device_count(), 4)
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), str(ROOT / "tests" / "step_dp_check.py")],
                       capture_output=True, text=True, timeout=600)
    print(p.stdout[-3000:])
    assert p.returncode == 0 and "STEP_DP_CHECK PASS" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]


def test_executor_data_parallel_path_single_gpu():
    """tests/step_dp_check.py at world 1: the executor's data-parallel schedule (per-key
    all-reduce on the comm stream, then the sharded optimizer's reduce-scatter / row-shard
    AdamW / all-gather + transpose) runs over a 1-rank NCCL communicator on one GPU — the
    driver's 1-GPU suite covers that code path, not only the >= 2-GPU runs."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=1", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), str(ROOT / "tests" / "step_dp_check.py")],
                       capture_output=True, text=True, timeout=600)
    print(p.stdout[-3000:])
    assert p.returncode == 0 and "STEP_DP_CHECK PASS" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]


def test_traced_step_timeline():
    """TLORA_RUN_TRACE: every op of the schedule gets its completion time on its own stream;
    times are ordered along each stream, cross-stream waits are respected (a GRADS op ends
    after the dX launch it waited for), and nothing ends after the step's end event."""
    from paper_2602_07263_b200 import capi
    ex = TrainingStep(MINI, device=0, nano_fixed=2, graphs=True)
    ex.init_random(MINI.seed)
    ex.enable_optimizer()
    ex.run()
    s = ex.run(trace=True)
    assert not s.replayed_graph
    tr = ex.trace()
    assert len(tr) == len(ex.layers) * 2 * 2 + 1 + len(ex.layers) * 2 + len(ex.layers)
    last = {}
    for i, (op, ms) in enumerate(tr):
        assert 0.0 < ms <= s.ms + 1e-3
        if op["stream"] in last:
            assert ms >= last[op["stream"]] - 1e-3
        last[op["stream"]] = ms
        for w in (op["wait0"], op["wait1"]):
            if w >= 0:
                assert ms >= tr[w][1] - 1e-3
    assert {op["stream"] for op, _ in tr} == {capi.STREAM_MAIN, capi.STREAM_SIDE}


def test_tp_executor_matches_python_tp_driver_multi_gpu():
    """tests/tp_exec_check.py under torchrun (>= 2 GPUs): the C++ TP step == the Python TP
    driver (bitwise activations, gradients within fp32 reassociation)."""
    import socket
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs (run via gpurun --gpus 2)")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    n = min(torch.cuda.device_count(), 4)
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), str(ROOT / "tests" / "tp_exec_check.py")],
                       capture_output=True, text=True, timeout=900)
    print(p.stdout[-3000:])
    assert p.returncode == 0 and "TP_EXEC_CHECK PASS" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]


@pytest.mark.parametrize("script,env", [
    ("tp_exec_check.py", {"TP_NANO": "3"}),
    ("tp_check.py", {"TP_NANO": "3", "TP_FUSED_RS": "1"}),
])
def test_tp_data_paths_single_gpu(script, env):
    """The tensor-parallel data paths on ONE GPU (world 1, TLORA_TP_CE_SELF=1): copy-engine
    all-gathers / slot-sum reduce-scatters and the fused GEMM + reduce-scatter epilogue push
    into this rank's own buffers. tp_exec_check: the C++ TP step == the Python TP driver
    (bitwise activations); tp_check: the Python TP driver == the unsharded layer."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    e = dict(os.environ, TLORA_TP_CE_SELF="1", **env)
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=1", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), str(ROOT / "tests" / script)],
                       capture_output=True, text=True, timeout=900, env=e)
    print(p.stdout[-3000:])
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]


def _executor_vs_oracle(wl, nano):
    """One executor step of `wl` at N = nano against the double oracle with bf16-emulated
    intermediates (oracle/tlora_oracle.c: fused_forward / fused_backward, pinned to the
    reference's goldens) on the executor's own token -> slot map: per (layer, projection)
    the H stash and dA / dB of every job, the last layer's Y and layer 0's dX. Tolerances
    as SURVEY §8(c) / test_gpu_step_parity."""
    st = TrainingStep(wl, device=0, nano_fixed=nano, graphs=False)
    st.init_random(wl.seed, keep_weights=True)
    st.enable_optimizer()  # (the step's AdamW runs after the gradients this test reads)
    s = st.run()
    torch.cuda.synchronize()
    assert s.nano_used == min(nano, sum(j.batch for j in wl.jobs))
    n_used, t0, ns, _ = st.layout(nano)
    slots = np.full(st.T, -1, np.int32)
    for i in range(n_used):
        row = int(t0[i])
        for sl, j in enumerate(wl.jobs):
            rows = int(ns[i, sl]) * j.seq_len
            slots[row:row + rows] = sl
            row += rows
    assert (slots >= 0).all()
    f64 = lambda t: t.double().cpu().numpy()  # noqa: E731

    def check(what, got, ref, tol):
        got = np.asarray(got, np.float64)
        mx = np.abs(got - ref).max() / max(1.0, np.abs(ref).max())
        fr = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
        assert mx <= tol[0] and fr <= tol[1], (what, mx, fr)

    last = wl.layers - 1
    for key in st.keys:
        L, name = key
        lay = st.layers[key]
        W, ab = st.weights[key]
        X, dY = f64(st.X[0][INPUT_GROUP.get(name, name)]), f64(st.dY[0][name])
        A = [f64(a) for a, _ in ab]
        B = [f64(b) for _, b in ab]
        Y, H = O.fused_forward(X, f64(W), A, B, slots, round_bf16=True, want_h=True)
        dX, dA, dB = O.fused_backward(X, f64(W), A, B, slots, dY, round_bf16=True,
                                      want_dx=(L == 0))
        Hd = f64(st.H[key])
        cum = np.concatenate([[0], np.cumsum([j.rank for j in wl.jobs])])
        for sl, j in enumerate(wl.jobs):
            rows = slots == sl
            off = lay.offsets[sl]
            check(f"H {key} {sl}", Hd[rows, off:off + j.rank], H[rows, cum[sl]:cum[sl] + j.rank],
                  (1e-2, 4e-3))
            gA, gB = lay.read_grad(sl)
            check(f"dA {key} {sl}", f64(gA), dA[sl], (2e-2, 8e-3))
            check(f"dB {key} {sl}", f64(gB), dB[sl], (2e-2, 8e-3))
        if L == last:
            check(f"Y {name}", f64(st.Y[name]), Y, (1e-2, 4e-3))
        if L == 0:
            check(f"dX {name}", f64(st.dX[name]), dX, (1e-2, 4e-3))


def test_executor_layer_stack_vs_oracle():
    """A 2-layer x 4-projection stack (4 jobs, ranks 8-200, ragged T) through the executor
    at N = 3: nano-major layout, chained schedule, side-stream gradients."""
    _executor_vs_oracle(MINI, 3)


@pytest.mark.parametrize("cell,nano", [((1024, 8, 4096, 5), 3), ((2048, 16, 4096, 6), 4),
                                       ((1024, 32, 2048, 7), 5), ((2048, 12, 3000, 8), 1)])
def test_executor_c5_cells_vs_oracle(cell, nano):
    """C5 heterogeneity cells (ranks 4-256, Zipf-skewed ragged token counts, one sample per
    job) through the executor: the rank-aware map puts whole jobs into nano-batches."""
    from paper_2602_07263_b200.workload import c5_cell
    _executor_vs_oracle(c5_cell(*cell), nano)


def test_tail_split_knob_parity():
    """TLORA_TAIL_SPLIT=1 (off by default: split-K of each fused launch's last partial wave)
    keeps the benched C2 step inside the fp32-restatement tolerances and the executor
    bitwise equal to the Python driver (both see the same split tables). Subprocess: the
    knob is read once per process."""
    e = dict(os.environ, TLORA_TAIL_SPLIT="1")
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-x",
                        str(ROOT / "tests" / "test_gpu_step_parity.py") + "::test_c2_benched_step_full_size",
                        str(ROOT / "tests" / "test_gpu_executor.py") + "::test_executor_matches_python_driver_bitwise"],
                       capture_output=True, text=True, timeout=900, env=e, cwd=str(ROOT))
    print(p.stdout[-2000:])
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]


def _random_workload(seed):
    rs = np.random.RandomState(seed)
    nproj = int(rs.randint(1, 4))
    projs = []
    for name in [f"p{i}" for i in range(nproj)]:  # each its own input group
        d = int(rs.choice([64, 136, 256, 392, 512]))
        k = int(rs.choice([64, 200, 256, 512, 768]))
        projs.append((str(name), d, k))
    lim = min(min(d, k) for _, d, k in projs)
    jobs = []
    for j in range(int(rs.randint(1, 7))):
        r = int(min(lim, rs.choice([1, 3, 8, 16, 40, 64, 128, 200])))
        jobs.append(Job(f"r{j}", r, int(rs.randint(1, 4)), int(rs.choice([1, 7, 64, 128, 300]))))
    return Workload(f"rand{seed}", projs, jobs, layers=int(rs.randint(1, 3)), seed=seed)


@pytest.mark.parametrize("seed", range(int(os.environ.get("TLORA_RANDOM_CASES", "24"))))
def test_executor_random_workloads_vs_oracle(seed):
    """Seeded random layer sets (1-3 projections with d, k down to 64 and not multiples of
    64, 1-6 jobs with ranks 1-200, sequence lengths 1-300, 1-2 layers) through the
    executor at a random N (1-5, also above the sample count) against the double oracle."""
    wl = _random_workload(seed)
    nano = int(np.random.RandomState(1000 + seed).randint(1, 6))
    _executor_vs_oracle(wl, nano)
