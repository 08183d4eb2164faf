"""CPU baseline leg of bench.py (placeholder until oracle tools are built)."""


def measure(wl, tokens_per_job=4, seconds_budget=15.0, threads=1, repeats=1):
    return None
