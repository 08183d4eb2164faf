"""The measured B200 cost model as the reference planner consumes it
(include/lora_fleet/hardware.hpp, through tests/cpp/_build/cost_main): HardwareSpec fields
validate and carry the fitted rates, and the C++ prediction reproduces the fit of
profiles/b200_cost_profile.json on its own measured grid (same median error)."""
import json
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "tests" / "cpp" / "_build" / "cost_main"
PROFILE = ROOT / "profiles" / "b200_cost_profile.json"


def predict(cells):
    """cells: [(d, k, ranks, tokens_per_job_list)] -> (hardware spec, [seconds])"""
    if not BIN.exists():
        subprocess.run(["make", "-C", str(ROOT), "tests/cpp/_build/cost_main"], check=True)
    lines = "".join(f"{d} {k} {','.join(map(str, r))} {','.join(map(str, t))}\n"
                    for d, k, r, t in cells)
    p = subprocess.run([str(BIN), str(PROFILE)], input=lines, capture_output=True, text=True,
                       check=True)
    out = p.stdout.strip().splitlines()
    return json.loads(out[0]), [float(x) for x in out[1:]]


def test_hardware_spec_from_profile():
    prof = json.loads(PROFILE.read_text())
    spec, _ = predict([])
    assert spec["gpu_flops"] == float(f"{prof['F_flops_per_s']:.6e}")
    assert abs(spec["kernel_launch_overhead"] - prof["hardware_spec"]["kernel_launch_overhead"]) \
        <= 1e-6 * prof["hardware_spec"]["kernel_launch_overhead"]
    assert spec["intra_node_bw"] >= 5e8 and spec["backward_multiplier"] == 2.0


def test_prediction_reproduces_the_fit_on_its_grid():
    prof = json.loads(PROFILE.read_text())
    grid = prof["grid"]
    cells = [(g["d"], g["k"], g["ranks"], [g["T"] // g["jobs"]] * g["jobs"]) for g in grid]
    _, pred = predict(cells)
    errs = [abs(p - g["step_ms"] * 1e-3) / (g["step_ms"] * 1e-3) for p, g in zip(pred, grid)]
    assert abs(float(np.median(errs)) - prof["fit_rel_err_median"]) < 1e-6
    assert abs(float(np.max(errs)) - prof["fit_rel_err_max"]) < 1e-6
