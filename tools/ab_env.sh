#!/bin/bash
# A/B of one environment knob on the default bench, interleaved: ab_env.sh VAR "A B" REPS OUTDIR [bench args]
# Prints value / ms_per_step / clocks per run; JSON lines land in OUTDIR.
VAR=$1; VALS=$2; REPS=$3; OUT=$4; shift 4
mkdir -p "$OUT"
for r in $(seq 1 "$REPS"); do
  for v in $VALS; do
    env "$VAR=$v" python bench.py --no-cpu-baseline --steps 20 --warmup 5 --aimd-steps 0 "$@" > "$OUT/${VAR}_${v}_$r.log" 2>&1
    python - "$OUT/${VAR}_${v}_$r.log" "$VAR=$v" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"),
      (d.get("roofline") or {}).get("frac"), flush=True)
PY
  done
done
