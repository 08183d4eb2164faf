"""Host-side logic of the C++ step executor (no GPU): the rank-aware nano-batch map
(tlora_nano_assign) bit-exact against its oracle restatement, the op schedule's ordering
and hazard invariants (tlora_step_schedule_host), and a gloo world-2 run of the
data-parallel schedule's dataflow (gradient accumulation over nano-batches, per-key
all-reduce issued right after the key's last nano-batch, AdamW on the mean)."""
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as O  # noqa: E402

from paper_2602_07263_b200 import capi  # noqa: E402
from paper_2602_07263_b200.layer import partition  # noqa: E402
from paper_2602_07263_b200.step import nano_assign, sample_weights, schedule_host  # noqa: E402
from paper_2602_07263_b200.workload import config  # noqa: E402


def _cases():
    rs = np.random.RandomState(5)
    out = []
    for name in ("C1", "C2", "C3", "C4"):
        wl = config(name)
        out.append(([j.batch for j in wl.jobs], sample_weights(wl)))
    for _ in range(60):
        S = int(rs.randint(1, 33))
        batch = rs.randint(0, 9, S)
        if batch.sum() == 0:
            batch[0] = 1
        weight = rs.randint(0, 1 << 40, S) if rs.rand() < 0.5 else rs.randint(0, 4, S)
        out.append((batch.tolist(), weight.tolist()))
    return out


def test_nano_assign_matches_oracle_bit_exact():
    for batch, weight in _cases():
        total = sum(batch)
        for n in (1, 2, 3, 4, 7, 8, total, total + 3):
            got = nano_assign(batch, weight, n)
            want = O.nano_assign(batch, weight, n)
            assert got[0] == want[0] and got[1] == want[1], (batch, n)
            assert np.array_equal(got[2], want[2]) and np.array_equal(got[3], want[3]), (batch, n)
            # counts are exactly the reference's partition (nano_pipeline.hpp:51-60)
            assert (got[0], got[1]) == partition(total, n)
            assert np.array_equal(got[3].sum(axis=1), got[1])
            assert np.array_equal(got[3].sum(axis=0), batch)
            # each (nano, job) is one contiguous range of the job's samples, in nano order
            off = 0
            for s, b in enumerate(batch):
                seg = got[2][off:off + b]
                assert np.all(np.diff(seg) >= 0)
                off += b


def test_nano_assign_errors():
    with pytest.raises(ValueError):
        nano_assign([0, 0], [1, 1], 2)
    with pytest.raises(ValueError):
        nano_assign([1, 2], [1, 1], 0)


def test_nano_assign_balances_lora_work_better_than_job_order():
    """Rank-aware map vs round 1's job-order slicing: the heaviest nano-batch carries no
    more work, and on C2 / C3 strictly less for N in 2..8."""
    for name in ("C2", "C3"):
        wl = config(name)
        batch, weight = [j.batch for j in wl.jobs], sample_weights(wl)
        samples = [w for b, w in zip(batch, weight) for _ in range(b)]
        for n in range(2, 9):
            k, per, _, ns = nano_assign(batch, weight, n)
            lpt = max(int(np.dot(ns[i], weight)) for i in range(k))
            order, i0 = [], 0
            for c in per:
                order.append(sum(samples[i0:i0 + c]))
                i0 += c
            assert lpt <= max(order), (name, n)


def _check_schedule(ops, keys, n, ring, side, dp, early=False):
    idx = {}
    for i, o in enumerate(ops):
        idx.setdefault((o["kind"], o["key"], o["nano"]), []).append(i)
    for key in range(keys):
        for nano in range(n):
            assert len(idx[(capi.OP_FWD, key, nano)]) == 1
            assert len(idx[(capi.OP_DX, key, nano)]) == 1
            assert len(idx[(capi.OP_GRADS, key, nano)]) == 1
            g = ops[idx[(capi.OP_GRADS, key, nano)][0]]
            assert g["beta"] == (1 if nano > 0 else 0)
            assert g["stream"] == (capi.STREAM_SIDE if side else capi.STREAM_MAIN)
        adam = [i for i, o in enumerate(ops) if o["kind"] == capi.OP_ADAMW and o["key"] == key]
        assert len(adam) == 1
        last_grads = idx[(capi.OP_GRADS, key, n - 1)][0]
        assert adam[0] > last_grads
        if dp == 2:  # sharded optimizer: reduce-scatter -> AdamW (own rows) -> all-gather
            rs = [i for i, o in enumerate(ops) if o["kind"] == capi.OP_REDUCE_SCATTER and o["key"] == key]
            ag = [i for i, o in enumerate(ops) if o["kind"] == capi.OP_ALLGATHER and o["key"] == key]
            assert len(rs) == 1 and len(ag) == 1 and rs[0] < adam[0] < ag[0]
            assert ops[rs[0]]["wait0"] == last_grads
            assert ops[rs[0]]["stream"] == ops[adam[0]]["stream"] == ops[ag[0]]["stream"] == capi.STREAM_COMM
            assert not any(o["kind"] == capi.OP_ALLREDUCE for o in ops)
        elif dp:
            ar = [i for i, o in enumerate(ops) if o["kind"] == capi.OP_ALLREDUCE and o["key"] == key]
            assert len(ar) == 1 and ar[0] < adam[0] and ops[ar[0]]["wait0"] == last_grads
            assert ops[ar[0]]["stream"] == ops[adam[0]]["stream"] == capi.STREAM_COMM
            if key > 0:  # issued while the backward of the lower keys is still to run
                assert ar[0] < idx[(capi.OP_DX, key - 1, n - 1)][0]
    # shrink of (key, nano) — standalone or as secondary tiles — before FWD(key, nano)
    made = {}
    for i, o in enumerate(ops):
        if o["kind"] == capi.OP_SHRINK:
            made[(o["key"], o["nano"])] = i
        if o["sec_kind"] == capi.OP_SHRINK:
            made[(o["sec_key"], o["sec_nano"])] = i
    for key in range(keys):
        for nano in range(n):
            assert made[(key, nano)] < idx[(capi.OP_FWD, key, nano)][0]
    # dH ring: every slot write happens after the previous reader of the slot finished
    # (same stream earlier, or an explicit wait), and every reader reads the slot its dH was
    # written into by an earlier main-stream launch
    last_reader, written = {}, {}
    for i, o in enumerate(ops):
        if o["sec_kind"] == capi.OP_DH:
            s = o["sec_slot"]
            if s in last_reader:
                j = last_reader[s]
                assert ops[j]["stream"] == o["stream"] or o["wait0"] == j or o["wait1"] == j, (i, j)
            written[(o["sec_key"], o["sec_nano"])] = (s, i)
        if o["kind"] in (capi.OP_DX, capi.OP_GRADS):
            s, w = written[(o["key"], o["nano"])]
            assert o["slot"] == s and w < i
        if o["kind"] == capi.OP_GRADS:
            last_reader[o["slot"]] = i
            if side:
                dx = idx[(capi.OP_DX, o["key"], o["nano"])][0]
                # after the key's dX launch, or (early) after the launch that wrote its dH
                assert o["wait0"] == (written[(o["key"], o["nano"])][1] if early else dx)
    # main-stream fused launches: exactly 2 x keys x n, plus the step's first shrink
    main = [o for o in ops if o["stream"] == capi.STREAM_MAIN and o["kind"] != capi.OP_GRADS
            and o["kind"] != capi.OP_ADAMW]
    assert len(main) == 2 * keys * n + 1


@pytest.mark.parametrize("keys", [1, 2, 7, 14])
@pytest.mark.parametrize("n", [1, 2, 3])
def test_schedule_invariants(keys, n):
    for ring in (2, 3, 8):
        for side in (2, 1, 0):
            for dp in (0, 1, 2):
                ops = schedule_host(keys, n, ring, side, dp)
                _check_schedule(ops, keys, n, ring, bool(side), dp, early=side == 2)


# ---------------------------------------------------------------- gloo world-2 dataflow
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _layout(batch, seq, weight, n):
    k, per, sample_nano, ns = O.nano_assign(batch, weight, n)
    slots_of_nano = [np.concatenate([np.full(ns[i, s] * seq[s], s, np.int32)
                                     for s in range(len(batch))]) for i in range(k)]
    return k, slots_of_nano


def _adam(p, g, lr, wd):  # first AdamW step from zero moments (the executor's optimizer)
    m, v = 0.1 * g, 0.001 * g * g
    return p - lr * ((m / 0.1) / (np.sqrt(v / 0.001) + 1e-8) + wd * p)


def _problem(rank):
    rs = np.random.RandomState(100 + rank)
    batch, seq, ranks = [2, 1, 3], [4, 6, 2], [3, 5, 2]
    T = sum(b * s for b, s in zip(batch, seq))
    dims = [(12, 10), (10, 8)]  # two keys (one layer, two projections)
    X = [rs.randn(T, d) for d, _ in dims]
    dY = [rs.randn(T, k) for _, k in dims]
    return batch, seq, ranks, dims, X, dY


def _params(ranks, dims):
    rs = np.random.RandomState(7)  # identical on every replica
    W = [rs.randn(d, k) for d, k in dims]
    A = [[rs.randn(d, r) for r in ranks] for d, _ in dims]
    B = [[rs.randn(r, k) for r in ranks] for _, k in dims]
    return W, A, B


def _dp_worker(rank, world, port, n, q):
    import os

    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        batch, seq, ranks, dims, X, dY = _problem(rank)
        W, A, B = _params(ranks, dims)
        weight = [1, 5, 2]
        k, slots = _layout(batch, seq, weight, n)
        t0 = np.concatenate([[0], np.cumsum([len(s) for s in slots])])
        ops = schedule_host(len(dims), k, 8, True, True)
        grads = [[None, None] for _ in dims]
        out = [[None, None] for _ in dims]
        order = []
        for o in ops:  # one valid linearisation of the three streams: list order
            key, i = o["key"], o["nano"]
            if o["kind"] == capi.OP_GRADS:
                r0, r1 = t0[i], t0[i + 1]
                _, dA, dB = O.fused_backward(X[key][r0:r1], W[key], A[key], B[key], slots[i],
                                             dY[key][r0:r1], want_dx=False)
                if o["beta"] == 0:
                    grads[key] = [dA, dB]
                else:
                    grads[key] = [[a + b for a, b in zip(grads[key][0], dA)],
                                  [a + b for a, b in zip(grads[key][1], dB)]]
            elif o["kind"] == capi.OP_ALLREDUCE:
                order.append(("ar", key))
                flat = torch.from_numpy(np.concatenate([g.ravel() for g in grads[key][0] + grads[key][1]]))
                dist.all_reduce(flat)
                vals, off = flat.numpy(), 0
                for part in grads[key]:
                    for j, g in enumerate(part):
                        part[j] = vals[off:off + g.size].reshape(g.shape)
                        off += g.size
            elif o["kind"] == capi.OP_ADAMW:
                order.append(("adam", key))
                out[key] = [[_adam(p, g / world, 1e-2, 0.01) for p, g in zip(A[key], grads[key][0])],
                            [_adam(p, g / world, 1e-2, 0.01) for p, g in zip(B[key], grads[key][1])]]
        # single-process reference: full-batch gradients of both replicas' data, summed
        ref = []
        for key in range(len(dims)):
            sA = [np.zeros_like(a) for a in A[key]]
            sB = [np.zeros_like(b) for b in B[key]]
            for rr in range(world):
                bt, sq, _, _, Xr, dYr = _problem(rr)
                # the replica's buffer rows carry the executor's token layout for n
                sl = np.concatenate(_layout(bt, sq, weight, n)[1])
                _, dA, dB = O.fused_backward(Xr[key], W[key], A[key], B[key], sl, dYr[key],
                                             want_dx=False)
                sA = [a + b for a, b in zip(sA, dA)]
                sB = [a + b for a, b in zip(sB, dB)]
            ref.append([[_adam(p, g / world, 1e-2, 0.01) for p, g in zip(A[key], sA)],
                        [_adam(p, g / world, 1e-2, 0.01) for p, g in zip(B[key], sB)]])
        ok = True
        for key in range(len(dims)):
            for part in range(2):
                for a, b in zip(out[key][part], ref[key][part]):
                    ok &= bool(np.allclose(a, b, rtol=1e-9, atol=1e-12))
        # the all-reduce of the last key (backward runs keys in reverse) comes first
        ok &= order[0] == ("ar", len(dims) - 1)
        q.put((rank, ok, k))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1, 3])
def test_dp_nano_schedule_gloo_world2(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert all(k == n for _, _, k in res)
