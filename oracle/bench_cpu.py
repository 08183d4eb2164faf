"""CPU baseline leg of bench.py: the reference's CPU path timed on the host cores.
TEST / BASELINE INFRASTRUCTURE (lives with the oracle): imported only by bench.py's
cpu_baseline leg and its reference arm, never by the product package.

kind "reference": oracle/_ref/ref_harness bench — the UNMODIFIED reference fused_forward
(proj/include/lora_fleet/fused_lora.hpp:84-119, compiled against the Eigen-subset shim)
for the forward and, on the transposed problem, for dX; dA/dB with the shim GEMM (the
reference has no backward). Tokens are sharded over all host threads (the reference
functions are pure and reentrant).
kind "port": the C oracle (oracle/liboracle.so), when the reference harness is absent.
Only this module (bench.py's cpu_baseline / reference arm) may execute oracle/.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF = HERE / "_ref" / "ref_bench"


def _run_ref(wl, threads, tokens_per_job, repeats, min_seconds=0.0):
    projs = ";".join(f"{d}:{k}" for _, d, k in wl.projections)
    ranks = ",".join(str(r) for r in wl.ranks)
    out = subprocess.run([str(REF), "bench", str(threads), str(tokens_per_job), str(repeats),
                          ranks, projs, str(min_seconds)], check=True, capture_output=True,
                         text=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def _run_port(wl, threads, tokens_per_job, repeats, min_seconds=0.0):
    import numpy as np
    sys.path.insert(0, str(HERE))
    import oracle as O
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    rs = np.random.RandomState(2602)
    slots = np.repeat(np.arange(len(wl.jobs)), tokens_per_job).astype(np.int32)
    T = len(slots)
    P = []
    for _, d, k in wl.projections:
        P.append((rs.randn(d, k) / np.sqrt(d), [rs.randn(d, r) for r in wl.ranks],
                  [rs.randn(r, k) for r in wl.ranks], rs.randn(T, d), rs.randn(T, k)))
    per = []
    while len(per) < repeats or sum(per) < min_seconds:
        t0 = time.perf_counter()
        for W, A, B, X, dY in P:
            O.fused_forward(X, W, A, B, slots)
            O.fused_backward(X, W, A, B, slots, dY)
        per.append(time.perf_counter() - t0)
    return {"seconds": sum(per), "tokens": T * len(per), "threads": threads, "per_repeat": per,
            "repeats": len(per)}


def measure_oracle_f32(wl, tokens_per_job, seconds_budget=10.0, threads=None):
    """the repo's own oracle, fp32 fwd+bwd (orc_train_step_f32,
    cache-blocked, OpenMP over all host cores) over every projection of the workload on a
    job-contiguous sample of tokens_per_job tokens per job. One untimed warm-up, then
    repetitions until seconds_budget. Returns dict(value tokens/s, cores, sample, ...)."""
    import numpy as np
    threads = threads or os.cpu_count() or 1
    os.environ["OMP_NUM_THREADS"] = str(threads)  # read when liboracle first starts OpenMP
    sys.path.insert(0, str(HERE))
    import oracle as O
    rs = np.random.RandomState(2602)
    T = tokens_per_job * len(wl.jobs)
    off = np.arange(len(wl.jobs) + 1, dtype=np.int64) * tokens_per_job
    P = []
    for _, d, k in wl.projections:
        P.append(((rs.standard_normal((d, k)) / np.sqrt(d)).astype(np.float32),
                  [rs.standard_normal((d, r)).astype(np.float32) for r in wl.ranks],
                  [rs.standard_normal((r, k)).astype(np.float32) for r in wl.ranks],
                  rs.standard_normal((T, d)).astype(np.float32),
                  rs.standard_normal((T, k)).astype(np.float32)))

    def once():
        for W, A, B, X, dY in P:
            O.train_step_f32(X, W, A, B, off, dY)

    once()
    per = []
    while not per or sum(per) < seconds_budget:
        t0 = time.perf_counter()
        once()
        per.append(time.perf_counter() - t0)
    tokens = T * len(per)
    return {"value": round(tokens / sum(per), 3), "unit": "tokens/s", "cores": threads,
            "kind": "port", "dtype": "f32",
            "sample": (f"repo oracle orc_train_step_f32 (fp32 fwd+bwd, OpenMP, cache-blocked), "
                       f"{tokens_per_job} tokens/job x {len(wl.jobs)} jobs through all "
                       f"{len(wl.projections)} projections of {wl.name}, {len(per)} timed "
                       f"repetitions after 1 warm-up ({sum(per):.2f} s) on {threads} threads"),
            "tokens_per_thread": round(T / threads, 1)}


def measure(wl, tokens_per_job=4, seconds_budget=15.0, threads=None, repeats=1):
    """tokens/s of fwd+bwd over every projection of `wl` on a bounded token sample.
    With seconds_budget > 0, repeats are added until about that much CPU time is spent."""
    threads = threads or os.cpu_count() or 1
    kind = "reference" if REF.exists() else "port"
    run = _run_ref if kind == "reference" else _run_port
    try:
        res = run(wl, threads, tokens_per_job, max(1, repeats), seconds_budget)
    except Exception as e:  # pragma: no cover - reported, never silently replaced
        return {"value": None, "unit": "tokens/s", "cores": threads, "kind": kind,
                "sample": f"failed: {e}"}
    value = res["tokens"] / res["seconds"]
    tpt = tokens_per_job * len(wl.jobs) / threads
    sample = (f"{tokens_per_job} tokens/job x {len(wl.jobs)} jobs ({tpt:.0f} tokens per thread) through all "
              f"{len(wl.projections)} projections of {wl.name}, fwd+bwd, fp64, "
              f"{res['tokens']} tokens in {res['seconds']:.2f} s ({res.get('repeats', 1)} timed "
              f"repetitions after 1 warm-up, setup untimed) on {threads} threads"
              + (" (reference fused_forward for fwd and dX; shim GEMM for dA/dB)"
                 if kind == "reference" else " (C oracle port)"))
    return {"value": round(value, 3), "unit": "tokens/s", "cores": threads, "kind": kind,
            "sample": sample, "tokens": res["tokens"], "dtype": "f64", "tokens_per_thread": tpt,
            "per_repeat_s": res.get("per_repeat"), "tokens_per_repeat":
                res["tokens"] // max(1, res.get("repeats", 1))}
