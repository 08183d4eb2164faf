"""Short, ncu-friendly run of the benched training step (C2 through the C++ executor):
warm-up steps, then --steps eager steps (every kernel launched from the host, so ncu's
kernel filters and -s / -c counts see each launch). Not a benchmark: no numbers printed
here are bench values.

  python tools/prof_step.py [--config C2] [--steps 2] [--warmup 2] [--nano 1]
"""
import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2602_07263_b200.step import TrainingStep  # noqa: E402
from paper_2602_07263_b200.workload import config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--nano", type=int, default=1)
    ap.add_argument("--layers", type=int, default=0)
    a = ap.parse_args()
    wl = config(a.config)
    if a.layers:
        wl.layers = a.layers
    st = TrainingStep(wl, nano_fixed=a.nano, graphs=False)
    st.init_random()
    st.enable_optimizer()
    for _ in range(a.warmup + a.steps):
        s = st.run(eager=True)
    torch.cuda.synchronize()
    print(f"prof_step: {a.config} N={a.nano} last step {s.ms:.3f} ms, {s.launches} launches")


if __name__ == "__main__":
    main()
