#!/bin/bash
# Interleaved A/B/C... of environment settings on the default bench:
#   ab_multi.sh REPS OUTDIR "NAME1:VAR=a VAR2=b" "NAME2:VAR=c" ... [-- bench args]
REPS=$1; OUT=$2; shift 2
CFGS=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do CFGS+=("$1"); shift; done
[ "$1" == "--" ] && shift
mkdir -p "$OUT"
for r in $(seq 1 "$REPS"); do
  for c in "${CFGS[@]}"; do
    name=${c%%:*}; envs=${c#*:}
    env $envs python bench.py --no-cpu-baseline --steps 20 --warmup 5 --aimd-steps 0 "$@" > "$OUT/${name}_$r.log" 2>&1
    python - "$OUT/${name}_$r.log" "$name" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"),
      (d.get("roofline") or {}).get("frac"), flush=True)
PY
  done
done
