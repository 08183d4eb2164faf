"""ctypes wrapper of oracle/liboracle.so. TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg,
as the checker. See oracle/tlora_oracle.h for the contract and parity pinning.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lib = None

_D = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_I = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise ImportError(f"{LIB} not built: run `make` at the repo root")
        L = C.CDLL(str(LIB))
        PP = C.POINTER(C.POINTER(C.c_double))
        L.orc_fused_forward.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int32, _I, PP, PP,
                                        _D, _D, _I, C.c_int32, _D, C.c_void_p]
        L.orc_materialized.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int32, _I, PP, PP,
                                       _D, _D, _I, _D]
        L.orc_fused_backward.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int32, _I, PP, PP,
                                         _D, _D, _I, _D, C.c_int32, C.c_void_p, PP, PP]
        L.orc_op_cost.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                  np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS"), _I,
                                  C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                  C.POINTER(C.c_longlong)]
        L.orc_op_cost.restype = None
        L.orc_partition.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_int32), _I]
        L.orc_aimd_step.argtypes = [C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_double), C.c_int32, C.c_double, C.c_double,
                                    C.c_double]
        L.orc_plan_tiles.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int32, _I, _I, C.c_int32,
                                     C.c_void_p, C.c_int64]
        L.orc_plan_tiles.restype = C.c_int64
        L.orc_grad_schedule.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32,
                                        _I, _I]
        L.orc_grad_schedule.restype = C.c_int
        L.orc_nano_assign.argtypes = [C.c_int32, _I, np.ctypeslib.ndpointer(np.int64,
                                                                            flags="C_CONTIGUOUS"),
                                      C.c_int32, C.POINTER(C.c_int32), _I, _I, _I]
        L.orc_nano_assign.restype = C.c_int
        PF = C.POINTER(C.POINTER(C.c_float))
        _F = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
        L.orc_train_step_f32.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int32, _I,
                                         np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS"),
                                         _F, _F, PF, PF, _F, _F, _F, PF, PF]
        L.orc_train_step_f32.restype = None
        L.orc_round_bf16.argtypes = [C.c_double]
        L.orc_round_bf16.restype = C.c_double
        _lib = L
    return _lib


def _pp(mats):
    arr = (C.POINTER(C.c_double) * len(mats))()
    for i, m in enumerate(mats):
        arr[i] = m.ctypes.data_as(C.POINTER(C.c_double))
    return arr


def _c(a, dt=np.float64):
    return np.ascontiguousarray(a, dtype=dt)


def fused_forward(X, W, A, B, slots, round_bf16=False, want_h=False):
    """fused_lora.hpp:84-119. A/B lists in slot (std::map) order; slots int per token."""
    X, W = _c(X), _c(W)
    A = [_c(a) for a in A]
    B = [_c(b) for b in B]
    slots = _c(slots, np.int32)
    T, d = X.shape
    k = W.shape[1]
    ranks = np.array([a.shape[1] for a in A], np.int32)
    Y = np.empty((T, k))
    H = np.empty((T, int(ranks.sum()))) if want_h else None
    rc = lib().orc_fused_forward(T, d, k, len(A), ranks, _pp(A), _pp(B), X, W, slots,
                                 int(round_bf16), Y, None if H is None else H.ctypes.data)
    if rc != 0:
        raise RuntimeError("fused_lora: segment has no adapter")
    return (Y, H) if want_h else Y


def materialized(X, W, A, B, slots):
    """fused_lora.hpp:124-135."""
    X, W = _c(X), _c(W)
    A = [_c(a) for a in A]
    B = [_c(b) for b in B]
    slots = _c(slots, np.int32)
    T, d = X.shape
    k = W.shape[1]
    ranks = np.array([a.shape[1] for a in A], np.int32)
    Y = np.zeros((T, k))
    if lib().orc_materialized(T, d, k, len(A), ranks, _pp(A), _pp(B), X, W, slots, Y) != 0:
        raise RuntimeError("fused_lora: segment has no adapter")
    return Y


def fused_backward(X, W, A, B, slots, dY, round_bf16=False, want_dx=True):
    X, W, dY = _c(X), _c(W), _c(dY)
    A = [_c(a) for a in A]
    B = [_c(b) for b in B]
    slots = _c(slots, np.int32)
    T, d = X.shape
    k = W.shape[1]
    ranks = np.array([a.shape[1] for a in A], np.int32)
    dX = np.empty((T, d)) if want_dx else None
    dA = [np.empty_like(a) for a in A]
    dB = [np.empty_like(b) for b in B]
    rc = lib().orc_fused_backward(T, d, k, len(A), ranks, _pp(A), _pp(B), X, W, slots, dY,
                                  int(round_bf16), None if dX is None else dX.ctypes.data,
                                  _pp(dA), _pp(dB))
    if rc != 0:
        raise RuntimeError("fused_lora: segment has no adapter")
    return dX, dA, dB


def op_cost(T, d, k, tokens_per_slot, ranks, fused=True):
    f, b, l = C.c_double(), C.c_double(), C.c_longlong()
    lib().orc_op_cost(T, d, k, len(ranks), _c(tokens_per_slot, np.int64), _c(ranks, np.int32),
                      int(fused), C.byref(f), C.byref(b), C.byref(l))
    return f.value, b.value, l.value


def partition(group_batch, n):
    out_n = C.c_int32()
    buf = np.zeros(max(1, n), np.int32)
    if lib().orc_partition(group_batch, n, C.byref(out_n), buf) != 0:
        raise ValueError("partition: invalid argument")
    return out_n.value, buf[: out_n.value].tolist()


def aimd_step(n, t_prev, t, alpha=4, beta=0.5, tau_rel=0.0):
    nn, hp, tp = C.c_int32(n), C.c_int32(t_prev is not None), C.c_double(t_prev or 0.0)
    if lib().orc_aimd_step(C.byref(nn), C.byref(hp), C.byref(tp), alpha, beta, tau_rel, t) != 0:
        raise ValueError("aimd_step: invalid argument")
    return nn.value, tp.value


def plan_tiles(T, d, k, ranks, slots, which):
    ranks = _c(ranks, np.int32)
    slots = _c(slots, np.int32)
    n = lib().orc_plan_tiles(T, d, k, len(ranks), ranks, slots, which, None, 0)
    if n < 0:
        raise ValueError("plan oracle: invalid input")
    out = np.zeros((max(1, n), 8), np.int32)
    lib().orc_plan_tiles(T, d, k, len(ranks), ranks, slots, which, out.ctypes.data, n)
    return out[:n]


def grad_schedule(tiles_db, tiles_da, ctas):
    """LPT CTA tile lists of one dB+dA launch (orc_grad_schedule): (off[ctas+1], idx)."""
    db = _c(tiles_db, np.int32).reshape(-1, 8)
    da = _c(tiles_da, np.int32).reshape(-1, 8)
    off = np.zeros(ctas + 1, np.int32)
    idx = np.zeros(max(1, len(db) + len(da)), np.int32)
    if lib().orc_grad_schedule(db.ctypes.data, len(db), da.ctypes.data, len(da), ctas, off,
                               idx) != 0:
        raise ValueError("schedule oracle: invalid input")
    return off, idx[: len(db) + len(da)]


def round_bf16(a):
    """Vectorised bf16 RNE rounding (numpy restatement of orc_round_bf16)."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = ((u + 0x7FFF + lsb) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32).astype(np.float64)


def nano_assign(batch, weight, n):
    """Rank-aware sample -> nano-batch map (orc_nano_assign): (n, per_nano, sample_nano,
    nano_slot[n x S])."""
    batch = _c(batch, np.int32)
    weight = _c(weight, np.int64)
    S, total = len(batch), int(batch.sum())
    out_n = C.c_int32()
    per = np.zeros(max(1, min(max(n, 1), max(total, 1))), np.int32)
    sn = np.zeros(max(1, total), np.int32)
    ns = np.zeros(max(1, per.size * S), np.int32)
    if lib().orc_nano_assign(S, batch, weight, n, C.byref(out_n), per, sn, ns) != 0:
        raise ValueError("nano_assign: invalid argument")
    m = out_n.value
    return m, per[:m].tolist(), sn[:total], ns[: m * S].reshape(m, S)


def _ppf(mats):
    arr = (C.POINTER(C.c_float) * len(mats))()
    for i, m in enumerate(mats):
        arr[i] = m.ctypes.data_as(C.POINTER(C.c_float))
    return arr


def train_step_f32(X, W, A, B, offsets, dY):
    """fp32 fwd+bwd of one layer on a job-contiguous batch (orc_train_step_f32): the
    CPU baseline's timed body. Returns Y, dX, dA, dB (float32)."""
    X, W, dY = _c(X, np.float32), _c(W, np.float32), _c(dY, np.float32)
    A = [_c(a, np.float32) for a in A]
    B = [_c(b, np.float32) for b in B]
    T, d = X.shape
    k = W.shape[1]
    ranks = np.array([a.shape[1] for a in A], np.int32)
    Y = np.empty((T, k), np.float32)
    dX = np.empty((T, d), np.float32)
    dA = [np.empty_like(a) for a in A]
    dB = [np.empty_like(b) for b in B]
    lib().orc_train_step_f32(T, d, k, len(A), ranks, _c(offsets, np.int64), X, W, _ppf(A),
                             _ppf(B), dY, Y, dX, _ppf(dA), _ppf(dB))
    return Y, dX, dA, dB
