#!/bin/bash
# Same box: the fused GEMM compiled with / without the tail split-K epilogue code (off at
# run time in both): ncu DRAM bytes of one step's 14 fused launches, then bench A/B.
OUT=$1
mkdir -p "$OUT"
NS=$PWD/paper_2602_07263_b200/libtlora_nosplit.so
for v in with without; do
  envs=""; [ $v = without ] && envs="TLORA_LIB=$NS"
  env $envs timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:lora_gemm2 --launch-skip 31 -c 14 --csv \
    --log-file "$OUT/traffic_$v.csv" python tools/prof_step.py --warmup 2 --steps 1 > "$OUT/ncu_$v.log" 2>&1
  python - "$OUT/traffic_$v.csv" $v <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, rows = rows[0], rows[1:]
ii, mi, vi = h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
per = collections.defaultdict(dict)
for r in rows:
    per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
rd = sum(v["dram__bytes_read.sum"] for v in per.values()); wr = sum(v["dram__bytes_write.sum"] for v in per.values())
t = sum(v["gpu__time_duration.sum"] for v in per.values())
print(f"{sys.argv[2]}: DRAM read {rd/1e9:.2f} GB write {wr/1e9:.2f} GB per step, serialised {t/1e6:.3f} ms", flush=True)
PY
done
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
e = d.get("energy") or {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"), e.get("joules_per_step"), flush=True)
PY
}
for rep in 1 2 3; do
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --aimd-steps 0 > "$OUT/with_$rep.log" 2>&1; summ "$OUT/with_$rep.log" with_$rep
  TLORA_LIB=$NS python bench.py --steps 20 --warmup 5 --no-cpu-baseline --aimd-steps 0 > "$OUT/without_$rep.log" 2>&1; summ "$OUT/without_$rep.log" without_$rep
done
