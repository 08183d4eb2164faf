"""Reader for the golden-vector records written by oracle/ref_harness.cpp (golden mode).

Record layout (little endian): i32 d, k, S, T; per adapter i32 rank, i32 len, id bytes;
T x i32 adapter index; f64 W[d*k], X[T*d], per adapter A[d*r], B[r*k]; f64 Y_fused[T*k],
Y_mat[T*k]; f64 flops, bytes; i64 launches; f64 u_flops, u_bytes; i64 u_launches.
Matrices are row-major. Adapter order is the reference's vector order; `slot_order` maps
it to std::map-by-job_id order (fused_lora.hpp:48-53).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np


@dataclass
class GoldenInstance:
    d: int
    k: int
    job_ids: list
    ranks: list
    owner: np.ndarray        # adapter index (vector order) per token
    W: np.ndarray
    X: np.ndarray
    A: list
    B: list
    Y_fused: np.ndarray
    Y_mat: np.ndarray
    cost: tuple              # (flops, bytes, launches)
    unfused: tuple
    raw: bytes = b""

    @property
    def tokens(self) -> int:
        return int(self.owner.shape[0])

    def slot_order(self):
        """Adapter indices sorted by job_id (std::map order); last duplicate wins."""
        by_id = {}
        for i, j in enumerate(self.job_ids):
            by_id[j] = i
        return [by_id[j] for j in sorted(by_id)]


def read_records(buf: bytes):
    off = 0
    out = []
    while off < len(buf):
        start = off
        d, k, S, T = struct.unpack_from("<4i", buf, off)
        off += 16
        ids, ranks = [], []
        for _ in range(S):
            r, n = struct.unpack_from("<2i", buf, off)
            off += 8
            ids.append(buf[off:off + n].decode())
            off += n
            ranks.append(r)
        owner = np.frombuffer(buf, "<i4", T, off).copy()
        off += 4 * T

        def mat(rows, cols):
            nonlocal off
            m = np.frombuffer(buf, "<f8", rows * cols, off).reshape(rows, cols).copy()
            off += 8 * rows * cols
            return m

        W = mat(d, k)
        X = mat(T, d)
        A, B = [], []
        for r in ranks:
            A.append(mat(d, r))
            B.append(mat(r, k))
        Yf = mat(T, k)
        Ym = mat(T, k)
        fl, by = struct.unpack_from("<2d", buf, off)
        off += 16
        (la,) = struct.unpack_from("<q", buf, off)
        off += 8
        ufl, uby = struct.unpack_from("<2d", buf, off)
        off += 16
        (ula,) = struct.unpack_from("<q", buf, off)
        off += 8
        out.append(GoldenInstance(d, k, ids, ranks, owner, W, X, A, B, Yf, Ym, (fl, by, la),
                                  (ufl, uby, ula), buf[start:off]))
    return out
