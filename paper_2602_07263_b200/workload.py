"""Synthetic workloads of SURVEY.md §8(d) (configs C1-C5 of BASELINE.json).

A workload is a set of adapted projections sharing one ragged multi-job token batch.
Every projection is one FusedLoRALayer with its own frozen W and per-job adapters; a
training "step" is fwd of every projection, then bwd of every projection (no attention,
no activation: the layer is the unit of work).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# projection name -> (d_in, d_out)
QWEN3_8B = [("q", 4096, 4096), ("k", 4096, 1024), ("v", 4096, 1024), ("o", 4096, 4096),
            ("gate", 4096, 12288), ("up", 4096, 12288), ("down", 12288, 4096)]
LLAMA3_8B = [("q", 4096, 4096), ("k", 4096, 1024), ("v", 4096, 1024), ("o", 4096, 4096),
             ("gate", 4096, 14336), ("up", 4096, 14336), ("down", 14336, 4096)]
QWEN3_32B = [("q", 5120, 8192), ("k", 5120, 1024), ("v", 5120, 1024), ("o", 8192, 5120),
             ("gate", 5120, 25600), ("up", 5120, 25600), ("down", 25600, 5120)]
# which projections read the same activation (one X per group)
INPUT_GROUP = {"q": "attn_in", "k": "attn_in", "v": "attn_in", "o": "o_in",
               "gate": "mlp_in", "up": "mlp_in", "down": "down_in"}


@dataclass
class Job:
    job_id: str
    rank: int
    batch: int      # samples
    seq_len: int

    @property
    def tokens(self) -> int:
        return self.batch * self.seq_len


@dataclass
class Workload:
    name: str
    projections: list           # [(name, d, k)]
    jobs: list                  # [Job], in reference adapter order (sorted job_id)
    layers: int = 1
    notes: str = ""
    seed: int = 2602

    @property
    def tokens(self) -> int:
        return sum(j.tokens for j in self.jobs)

    @property
    def ranks(self) -> list:
        return [j.rank for j in self.jobs]

    def token_slots(self, shuffle: bool = False, seed: int | None = None) -> np.ndarray:
        """Job-contiguous owner slot per token (shuffled when asked, like
        test_fused_lora.cpp:46)."""
        slots = np.concatenate([np.full(j.tokens, s, np.int32) for s, j in enumerate(self.jobs)])
        if shuffle:
            np.random.RandomState(self.seed if seed is None else seed).shuffle(slots)
        return slots

    def flops_fwd_bwd(self) -> float:
        """Algorithmic FLOPs of one step: sum over projections and layers of
        4·T·d·k + 6·Σ_j T_j·r_j·(d+k) (no dW, W frozen)."""
        rt = sum(j.tokens * j.rank for j in self.jobs)
        T = self.tokens
        return self.layers * sum(4.0 * T * d * k + 6.0 * rt * (d + k)
                                 for _, d, k in self.projections)


def _sorted(jobs):
    return sorted(jobs, key=lambda j: j.job_id)  # std::map order, fused_lora.hpp:48-53


def config(name: str) -> Workload:
    name = name.upper()
    if name == "C1":
        jobs = [Job("j0", 8, 4, 512), Job("j1", 16, 1, 512), Job("j2", 32, 8, 512),
                Job("j3", 64, 2, 512)]
        return Workload("C1", [("proj", 1024, 1024)], _sorted(jobs), seed=2602 + 1,
                        notes="single SSM linear layer d=k=1024, 4 jobs r={8,16,32,64}")
    if name == "C2":
        ranks = [8, 16, 24, 32, 48, 64, 96, 128]
        batches = [1, 2, 1, 4, 2, 1, 4, 1]
        jobs = [Job(f"job{i}", r, b, 1024) for i, (r, b) in enumerate(zip(ranks, batches))]
        return Workload("C2", QWEN3_8B, _sorted(jobs), seed=2602 + 2,
                        notes="Qwen3-8B q/k/v/o/gate/up/down, 8 jobs r=8..128, T=16384")
    if name == "C3":
        ranks = [8, 16, 32, 64, 128, 24, 48, 96] * 2
        batches = [1, 2, 4, 8] * 4
        jobs = [Job(f"job{i:02d}", r, b, 1024) for i, (r, b) in enumerate(zip(ranks, batches))]
        return Workload("C3", LLAMA3_8B, _sorted(jobs), layers=32, seed=2602 + 3,
                        notes="Llama-3-8B 32 layers x 7 projections, 16 jobs, T=61440/replica")
    if name == "C4":
        ranks = [8, 16, 32, 64, 128, 24, 48, 96] * 2
        batches = [1, 2, 4, 8] * 4
        jobs = [Job(f"job{i:02d}", r, b, 1024) for i, (r, b) in enumerate(zip(ranks, batches))]
        return Workload("C4", QWEN3_32B, _sorted(jobs), layers=64, seed=2602 + 4,
                        notes="Qwen3-32B 64 layers, TP over W")
    raise KeyError(name)


def c5_cell(d: int, n_jobs: int, total_tokens: int, seed: int) -> Workload:
    """One cell of the C5 heterogeneity sweep: ranks in [4, 256], Zipf(1.2)-skewed batch."""
    rs = np.random.RandomState(seed)
    pool = [4, 8, 12, 16, 24, 40, 64, 100, 128, 200, 256]
    ranks = [int(rs.choice(pool)) for _ in range(n_jobs)]
    w = 1.0 / np.arange(1, n_jobs + 1) ** 1.2
    w = w / w.sum()
    counts = np.maximum(1, np.floor(w * total_tokens)).astype(int)
    counts[0] += total_tokens - counts.sum()
    jobs = [Job(f"j{i:02d}", min(r, d), 1, int(c)) for i, (r, c) in enumerate(zip(ranks, counts))]
    return Workload(f"C5[d={d},J={n_jobs},T={total_tokens},s={seed}]", [("proj", d, d)],
                    _sorted(jobs), seed=seed)
