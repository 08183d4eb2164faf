"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of the bench: per
kernel, launches and serialised time per step, and each kernel's share of the step.

  python tools/launch_summary.py launches.csv LAUNCHES_PER_STEP
"""
import collections
import csv
import re
import sys


def main():
    path, per_step = sys.argv[1], int(sys.argv[2])
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    ks = [(re.sub(r"\(.*", "", r[ki]).replace("void ", ""), float(r[vi].replace(",", "")))
          for r in rows]
    steps = len(ks) // per_step
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for name, ns in ks[: steps * per_step]:
        tot[name] += ns
        cnt[name] += 1
    step_ns = sum(tot.values()) / steps
    print(f"{len(ks)} launches = {steps} steps x {per_step}; serialised kernel time per step "
          f"{step_ns / 1e6:.3f} ms (ncu, --clock-control none, one kernel at a time)\n")
    print("| kernel | launches / step | ms / step | share |")
    print("|---|---|---|---|")
    for name in sorted(tot, key=lambda n: -tot[n]):
        print(f"| `{name}` | {cnt[name] / steps:g} | {tot[name] / steps / 1e6:.3f} | "
              f"{tot[name] / steps / step_ns:.3f} |")


if __name__ == "__main__":
    main()
