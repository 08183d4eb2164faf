"""CPU tests of the C-ABI boundary (no compute calls without a GPU).

 * libtlora.so loads and exports every entry point include/tlora.h declares;
 * the host-side reference restatements behind the ABI (OpCost, partition, aimd_step)
   are bit-identical to the reference golden values;
 * the rank-aware tile plan is bit-identical to the plan oracle (oracle/tlora_oracle.c);
 * without an sm_100 device, compute entry points fail loudly (no CPU fallback).
"""
import ctypes as C
import json
import re
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
import oracle as O  # noqa: E402
from golden_io import read_records  # noqa: E402

from paper_2602_07263_b200 import capi  # noqa: E402
from paper_2602_07263_b200.layer import (AimdState, aimd_step, op_cost, partition,  # noqa: E402
                                         grad_schedule_host, plan_tiles_host)
from paper_2602_07263_b200.workload import c5_cell, config  # noqa: E402
from conftest import has_gpu  # noqa: E402

KAT = json.loads((ROOT / "tests" / "golden" / "kat.json").read_text())


def header_symbols():
    text = (ROOT / "include" / "tlora.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int|long long)\s+(tlora_\w+)\(", text,
                                 re.M)))


def test_library_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 20
    lib = capi.lib()
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(capi.SIGNATURES), set(syms) ^ set(capi.SIGNATURES)
    assert lib.tlora_abi_version() == 5


def test_op_cost_via_abi_matches_reference_golden():
    for name in ("fused_2024.bin", "fused_99.bin"):
        for inst in read_records((ROOT / "tests" / "golden" / name).read_bytes()):
            order = inst.slot_order()
            pos = {a: s for s, a in enumerate(order)}
            slots = np.array([pos[a] for a in inst.owner])
            ranks = [inst.ranks[a] for a in order]
            tps = np.bincount(slots, minlength=len(ranks))
            assert op_cost(inst.tokens, inst.d, inst.k, tps, ranks, True) == inst.cost
            assert op_cost(inst.tokens, inst.d, inst.k, tps, ranks, False) == inst.unfused
    assert op_cost(2, 3, 2, [2], [1])[0] == 44.0


def test_partition_and_aimd_via_abi():
    for c in KAT["partition"]:
        assert partition(c["batch"], c["n"]) == (c["out_n"], c["per_nano"])
    with pytest.raises(ValueError):
        partition(0, 1)
    with pytest.raises(ValueError):
        partition(4, 0)
    for key, tau in (("aimd_tau0", 0.0), ("aimd_tau01", 0.1)):
        s = AimdState(n=8, tau_rel=tau)
        for t, expect in KAT[key]:
            s = aimd_step(s, t)
            assert s.n == expect
    with pytest.raises(ValueError):
        aimd_step(AimdState(n=1, t_prev=1.0), -1.0)
    with pytest.raises(ValueError):
        aimd_step(AimdState(beta=1.0), 1.0)


def _plan_cases():
    rs = np.random.RandomState(5)
    cases = []
    for shuffle in (False, True):
        for wl in (config("C1"), c5_cell(1024, 8, 2048, 3), c5_cell(4096, 32, 8192, 1)):
            cases.append((wl.projections[0][1], wl.projections[0][2], wl.ranks,
                          wl.token_slots(shuffle=shuffle)))
    # ragged / edge cases: 1 token, slots absent from the batch, rank 1 and 256
    cases.append((64, 8, [1], np.zeros(1, np.int32)))
    cases.append((256, 264, [4, 256, 8, 1], np.array([1] * 300 + [3] * 5, np.int32)))
    cases.append((128, 128, [16] * 40, rs.randint(0, 40, 1000).astype(np.int32)))
    c2 = config("C2")
    cases.append((4096, 12288, c2.ranks, c2.token_slots()))
    return cases


@pytest.mark.parametrize("case", range(len(_plan_cases())))
def test_plan_bit_identical_to_plan_oracle(case):
    d, k, ranks, slots = _plan_cases()[case]
    for launch in range(8):
        got = plan_tiles_host(d, k, ranks, slots, launch)
        want = O.plan_tiles(len(slots), d, k, ranks, slots, launch)
        assert got.shape == want.shape, (launch, got.shape, want.shape)
        assert np.array_equal(got, want), launch


@pytest.mark.parametrize("case", range(len(_plan_cases())))
def test_grad_schedule_bit_identical_to_schedule_oracle(case):
    """The LPT CTA tile lists the plan uploads for its dB+dA launch equal the oracle's
    restatement of the rule (cost, order, tie-breaks) for 148 CTAs and a small grid; every
    tile is scheduled exactly once."""
    d, k, ranks, slots = _plan_cases()[case]
    db = O.plan_tiles(len(slots), d, k, ranks, slots, capi.L_DB)
    da = O.plan_tiles(len(slots), d, k, ranks, slots, capi.L_DA)
    for ctas in (148, 7):
        off, idx = grad_schedule_host(d, k, ranks, slots, ctas)
        want_off, want_idx = O.grad_schedule(db, da, ctas)
        assert np.array_equal(off, want_off) and np.array_equal(idx, want_idx)
        assert np.array_equal(np.sort(idx), np.arange(len(db) + len(da)))


def test_grad_schedule_balances_c2():
    """On every C2 projection the busiest CTA carries <= 1.15x the mean bytes (round-robin
    over the largest-first list: 1.31-1.53x)."""
    c2 = config("C2")
    slots = c2.token_slots()
    for _, d, k in c2.projections:
        tiles = np.concatenate([plan_tiles_host(d, k, c2.ranks, slots, capi.L_DB),
                                plan_tiles_host(d, k, c2.ranks, slots, capi.L_DA)])
        cost = ((tiles[:, 3] - tiles[:, 2]).astype(np.int64) * 2 * (128 + (tiles[:, 7] + 63) // 64 * 64)
                + 4 * 128 * tiles[:, 7].astype(np.int64))
        off, idx = grad_schedule_host(d, k, c2.ranks, slots, 148)
        load = np.array([cost[idx[off[c]:off[c + 1]]].sum() for c in range(148)])
        assert load.max() <= 1.15 * load.mean()


def test_plan_covers_every_owned_column():
    """Size-independent property: every token's own packed rank columns lie inside the
    K-extension window of its M-tile, and windows are at most one K-block wider per side."""
    for d, k, ranks, slots in _plan_cases():
        off = np.concatenate([[0], np.cumsum([(r + 7) // 8 * 8 for r in ranks])])[:-1]
        fwd = plan_tiles_host(d, k, ranks, slots, capi.L_FWD)
        win = {int(t[0]): (int(t[4]), int(t[5])) for t in fwd}
        for m0, (lo, hi) in win.items():
            owned = slots[m0:m0 + 256]  # fused GEMMs run on 256-token CTA-pair tiles
            need_lo = min(off[s] for s in owned)
            need_hi = max(off[s] + ranks[s] for s in owned)
            assert lo <= need_lo and hi >= need_hi
            assert need_lo - lo < 64 and hi - need_hi < 64


def test_plan_rejects_unknown_slot():
    with pytest.raises(capi.TloraError) as e:
        plan_tiles_host(64, 64, [4, 4], [0, 1, 2], capi.L_FWD)
    assert e.value.code == capi.ERR_REGISTRY
    assert "no adapter" in str(e.value)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_device():
    from paper_2602_07263_b200.layer import FusedLoRALayer
    with pytest.raises(capi.TloraError) as e:
        FusedLoRALayer(64, 64, [4])
    assert e.value.code in (capi.ERR_NO_DEVICE, capi.ERR_CUDA)
    code = capi.lib().tlora_device_check(0, None)
    assert code in (capi.ERR_NO_DEVICE, capi.ERR_CUDA)


def test_shape_errors_are_status_codes():
    rk = (C.c_int32 * 1)(4)
    h = C.c_void_p()
    code = capi.lib().tlora_layer_create(0, 12, 64, 1, rk, C.byref(h))
    assert code == capi.ERR_SHAPE and "multiples of 8" in capi.lib().tlora_last_error().decode()
    rk = (C.c_int32 * 1)(0)
    code = capi.lib().tlora_layer_create(0, 64, 64, 1, rk, C.byref(h))
    assert code == capi.ERR_SHAPE


def test_profile_end_writes_exactly_prof_kinds_entries():
    """tlora_profile_end fills TLORA_PROF_KINDS entries per array (launch kinds 6/7, the
    secondary SHRINK2 / DH2 tiles, are booked under FWD / DX and have no slot)."""
    kinds = int(re.search(r"#define TLORA_PROF_KINDS (\d+)",
                          (ROOT / "include" / "tlora.h").read_text()).group(1))
    assert kinds == 6
    cnt = (C.c_int32 * (kinds + 2))(*([-7] * (kinds + 2)))
    ms = (C.c_double * (kinds + 2))(*([-7.0] * (kinds + 2)))
    fl = (C.c_double * (kinds + 2))(*([-7.0] * (kinds + 2)))
    assert capi.lib().tlora_profile_begin() == 0
    assert capi.lib().tlora_profile_end(cnt, ms, fl) == 0
    assert list(cnt[:kinds]) == [0] * kinds and list(ms[:kinds]) == [0.0] * kinds
    assert list(cnt[kinds:]) == [-7, -7] and list(ms[kinds:]) == [-7.0, -7.0]
    assert list(fl[kinds:]) == [-7.0, -7.0]


def test_segments_match_reference_segment_rows():
    """tlora_segments == detail::segment_rows (fused_lora.hpp:56-61: ascending rows whose
    segment_map entry is the job id) for every job, on the reference's own golden batches
    (shuffled segment maps, test_fused_lora.cpp:45-46) — bit-exact index lists."""
    from paper_2602_07263_b200.layer import segments
    n = 0
    for name in ("fused_2024.bin", "fused_101.bin"):
        for inst in read_records((ROOT / "tests" / "golden" / name).read_bytes()):
            order = inst.slot_order()
            slot_of_adapter = {a: s for s, a in enumerate(order)}
            ids = [inst.job_ids[a] for a in order]
            owner_ids = [inst.job_ids[a] for a in inst.owner]
            slots = np.array([slot_of_adapter[order[ids.index(j)]] for j in owner_ids], np.int32)
            perm, off = segments(slots, len(order))
            for s, jid in enumerate(ids):
                ref_rows = [t for t, j in enumerate(owner_ids) if j == jid]  # segment_rows
                assert perm[off[s]:off[s + 1]].tolist() == ref_rows
            n += 1
    assert n > 0
    with pytest.raises(capi.TloraError):
        segments(np.array([0, 3], np.int32), 2)
