#!/bin/bash
# Every bench.py variant a user may call still runs and prints a JSON line (1 GPU).
OUT=$1
mkdir -p "$OUT"
run() { local name=$1; shift; timeout 600 python bench.py "$@" > "$OUT/$name.log" 2>&1; echo "$name rc=$? $(grep -h '^{' "$OUT/$name.log" | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read() or "{}"); print(d.get("value"), d.get("ms_per_step"), (d.get("run") or d.get("config") or {}).get("driver"))' 2>&1)"; }
run host_cpp --host cpp --steps 5 --warmup 3 --no-cpu-baseline
run driver_py --driver python --steps 5 --warmup 3 --no-cpu-baseline
run aimd_timed --nano-batches 0 --steps 8 --warmup 3 --no-cpu-baseline
run c3_2layers --config C3 --layers 2 --steps 3 --warmup 3 --no-cpu-baseline
run c4_layer --config C4 --layers 1 --steps 3 --warmup 3 --no-cpu-baseline
run shuffled --shuffle --steps 5 --warmup 3 --no-cpu-baseline
