"""Tensor-parallel / nano-batch host logic on CPU (gloo, world_size 2), and the multi-GPU
parity check (tests/tp_check.py) when >= 2 GPUs are visible."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as O  # noqa: E402

from paper_2602_07263_b200.tp import nano_batches, shard_columns, shard_rows  # noqa: E402
from paper_2602_07263_b200.workload import config  # noqa: E402


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
@pytest.mark.parametrize("n", [1, 3, 4, 7, 16, 1000])
def test_nano_batches_follow_reference_partition(name, n):
    wl = config(name)
    nb = nano_batches(wl, n)
    total = sum(j.batch for j in wl.jobs)
    n_ref, counts = O.partition(total, n)  # nano_pipeline.hpp:51-60 (oracle)
    assert len(nb) == n_ref
    seq = {j.seq_len for j in wl.jobs}.pop()
    assert [b.tokens for b in nb] == [c * seq for c in counts]
    # whole samples, the rank-aware map (oracle restatement): nano i holds ns[i, s] samples
    # of job s, jobs in slot order
    from paper_2602_07263_b200.step import sample_weights
    _, _, _, ns = O.nano_assign([j.batch for j in wl.jobs], sample_weights(wl), n)
    for i, b in enumerate(nb):
        want = np.concatenate([np.full(ns[i, s] * j.seq_len, s, np.int32)
                               for s, j in enumerate(wl.jobs)])
        assert np.array_equal(b.slots, want)
    assert np.array_equal(np.sort(np.concatenate([b.slots for b in nb])), wl.token_slots())
    assert [b.t0 for b in nb] == list(np.cumsum([0] + [b.tokens for b in nb])[:-1])
    for b in nb:  # job-contiguous inside each nano-batch
        assert np.all(np.diff(b.slots) >= 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = config("C2")
        ok = True
        # sequence-parallel shards of every nano-batch re-assemble the nano-batch
        for b in nano_batches(wl, 5):
            r0, rows = b.shard(rank, world)
            mine = torch.from_numpy(b.slots[r0:r0 + rows].copy())
            parts = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(parts, mine)
            ok &= bool(torch.equal(torch.cat(parts), torch.from_numpy(b.slots)))
        # column / row weight shards re-assemble the full weight (all_gather = the TP AG)
        g = torch.Generator().manual_seed(0)
        W = torch.randn(64, 96, generator=g)
        c = shard_columns(W, rank, world)
        parts = [torch.empty_like(c) for _ in range(world)]
        dist.all_gather(parts, c)
        ok &= bool(torch.equal(torch.cat(parts, 1), W))
        r = shard_rows(W, rank, world)
        parts = [torch.empty_like(r) for _ in range(world)]
        dist.all_gather(parts, r)
        ok &= bool(torch.equal(torch.cat(parts, 0), W))
        # row-parallel identity the driver relies on: sum_p X_p W_p == X W (reduce-scatter)
        X = torch.randn(8, 64, generator=g, dtype=torch.float64)
        Wd = W.double()
        part = X[:, rank * 64 // world:(rank + 1) * 64 // world] @ shard_rows(Wd, rank, world)
        dist.all_reduce(part)
        ok &= bool(torch.allclose(part, X @ Wd, atol=1e-12))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_tp_sharding_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


@pytest.mark.gpu
def test_tp_parity_multi_gpu():
    # every visible GPU up to 4; on a 1-GPU box the NCCL all-gather / reduce-scatter path
    # at world 1 (the copy-engine and fused paths: test_tp_data_paths_single_gpu)
    n = max(1, min(torch.cuda.device_count(), 4))
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
                        "--master-port", str(_free_port()), str(ROOT / "tests" / "tp_check.py")],
                       capture_output=True, text=True, timeout=900)
    print(p.stdout[-3000:])
    assert p.returncode == 0 and "TP_CHECK PASS" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]


def test_monitor_restates_reference():
    """monitor() == nano_pipeline.hpp:114-126 on hand-built traces, including the degenerate
    ones (zero event time, zero stages)."""
    from paper_2602_07263_b200.layer import monitor
    eta, stall = monitor([1.0, 2.0, 3.0], [0.5, 0.5, 0.5], 8.0, 6.0, num_stages=2)
    assert eta == 6.0 / 16.0 and stall == 2.0
    assert monitor([1.0], [1.0], 0.0, 1.0) == (0.0, -1.0)
    assert monitor([1.0], [1.0], 2.0, 1.0, num_stages=0) == (0.0, 1.0)
