"""The measured cost model (include/lora_fleet/hardware.hpp, fitted by tools/cost_profile.py
on uniform job batches) predicting C5 heterogeneity cells it was NOT fitted on: skewed
Zipf(1.2) token counts, 2-32 jobs, ranks 4-256, d = k in {1024, 4096}. Measured: one
training step (fwd + bwd + fused AdamW) of the fused layer, CUDA events, mean of 10.
Stated bound: median relative error <= 15%, every cell <= 45% (small cells are launch-
bound and the model's fixed overheads are a fit average)."""
import numpy as np
import pytest
import torch

from paper_2602_07263_b200.layer import FusedLoRALayer
from paper_2602_07263_b200.workload import c5_cell
from test_cost_model import predict

pytestmark = pytest.mark.gpu


def _measure(d, ranks, counts, reps=10):
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(d + len(ranks))
    lay = FusedLoRALayer(d, d, ranks)
    lay.set_base((torch.randn(d, d, generator=g, device=dev) * d ** -0.5).bfloat16())
    for s, r in enumerate(ranks):
        lay.set_adapter(s, (torch.randn(d, r, generator=g, device=dev) * d ** -0.5).bfloat16(),
                        (torch.randn(r, d, generator=g, device=dev) * r ** -0.5).bfloat16())
    lay.set_optimizer(1e-4)
    slots = np.repeat(np.arange(len(ranks)), counts).astype(np.int32)
    T = len(slots)
    plan = lay.plan(slots)
    X = torch.randn(T, d, generator=g, device=dev).bfloat16()
    dY = torch.randn(T, d, generator=g, device=dev).bfloat16()
    Y = torch.empty(T, d, dtype=torch.bfloat16, device=dev)
    H = torch.zeros(T, lay.R, dtype=torch.bfloat16, device=dev)
    dX = torch.empty(T, d, dtype=torch.bfloat16, device=dev)

    def step():
        lay.forward(plan, X, Y, H)
        lay.backward(plan, dY, X, H, dX)
        lay.optimizer_step()

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    lay.close()
    return e0.elapsed_time(e1) / reps * 1e-3


def test_cost_model_predicts_c5_cells():
    cells, measured = [], []
    for d in (1024, 4096):
        for J in (2, 8, 32):
            for T in (2048, 8192):
                wl = c5_cell(d, J, T, seed=J + T)
                counts = [j.tokens for j in wl.jobs]
                cells.append((d, d, wl.ranks, counts))
                measured.append(_measure(d, wl.ranks, counts))
    _, pred = predict(cells)
    errs = [abs(p - m) / m for p, m in zip(pred, measured)]
    for (d, _, r, c), m, p, e in zip(cells, measured, pred, errs):
        print(f"d={d} J={len(r)} T={sum(c)}: measured {m * 1e3:.3f} ms, predicted "
              f"{p * 1e3:.3f} ms, err {e:.3f}")
    print(f"median err {np.median(errs):.3f}, max {np.max(errs):.3f}")
    assert np.median(errs) <= 0.15 and max(errs) <= 0.45
