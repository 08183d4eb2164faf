#!/bin/bash
# Tail split-K (TLORA_TAIL_SPLIT=1): parity of the benched step with it on, then an
# interleaved bench A/B against the default.  usage: tail_split_ab.sh OUTDIR
OUT=$1
mkdir -p "$OUT"
TLORA_TAIL_SPLIT=1 TLORA_TAIL_SPLIT_DEBUG=1 python tools/prof_step.py --warmup 1 --steps 1 > "$OUT/debug.log" 2>&1; grep tail_split "$OUT/debug.log" | sort | uniq | head -20
TLORA_TAIL_SPLIT=1 python -m pytest tests/test_gpu_step_parity.py tests/test_gpu_executor.py tests/test_gpu_parity.py -q -m gpu -x > "$OUT/tests_split.log" 2>&1; tail -2 "$OUT/tests_split.log"
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
r = d.get("roofline") or {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"), r.get("frac"), flush=True)
PY
}
for rep in 1 2 3; do
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --aimd-steps 0 > "$OUT/base_$rep.log" 2>&1; summ "$OUT/base_$rep.log" base_$rep
  TLORA_TAIL_SPLIT=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --aimd-steps 0 > "$OUT/split_$rep.log" 2>&1; summ "$OUT/split_$rep.log" split_$rep
done
