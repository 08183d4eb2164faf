#!/bin/bash
# Re-sweep of the fused GEMM's L2 panel budget at HEAD: ncu DRAM bytes of the 14 fused
# launches of one step, then bench step time / clock / energy per budget (interleaved).
OUT=$1
mkdir -p "$OUT"
for b in 16 24 32 48 64; do
  TLORA_L2_BUDGET_MB=$b timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:lora_gemm2 --launch-skip 31 -c 14 --csv \
    --log-file "$OUT/traffic_$b.csv" python tools/prof_step.py --warmup 2 --steps 1 > "$OUT/ncu_$b.log" 2>&1
  python - "$OUT/traffic_$b.csv" $b <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, rows = rows[0], rows[1:]
ii, mi, vi = h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
per = collections.defaultdict(dict)
for r in rows:
    per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
rd = sum(v["dram__bytes_read.sum"] for v in per.values()); wr = sum(v["dram__bytes_write.sum"] for v in per.values())
t = sum(v["gpu__time_duration.sum"] for v in per.values())
print(f"budget {sys.argv[2]} MB: {len(per)} launches, DRAM read {rd/1e9:.2f} GB write {wr/1e9:.2f} GB per step, serialised {t/1e6:.3f} ms", flush=True)
PY
done
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
e = d.get("energy") or {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"), e.get("joules_per_step"), e.get("avg_power_w"), flush=True)
PY
}
for rep in 1 2; do
  for b in 48 24 32 64; do
    TLORA_L2_BUDGET_MB=$b python bench.py --steps 20 --warmup 5 --no-cpu-baseline --aimd-steps 0 > "$OUT/bench_${b}_$rep.log" 2>&1; summ "$OUT/bench_${b}_$rep.log" "b${b}_$rep"
  done
done
