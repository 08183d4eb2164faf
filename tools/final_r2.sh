#!/bin/bash
# Round-2 closing evidence on one B200: the GPU test suite, smoke(), the default bench line,
# the reference arm, and the ncu launch list of the bench's own kernels (after the bench
# exited 0 without ncu).  usage: final_r2.sh OUTDIR
OUT=$1
mkdir -p "$OUT"
( time python -m pytest tests -q -m gpu -x ) > "$OUT/gpu_tests.log" 2>&1; tail -4 "$OUT/gpu_tests.log"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke OK')" > "$OUT/smoke.log" 2>&1; tail -1 "$OUT/smoke.log"
python bench.py --gpus 1 --steps 20 --warmup 5 > "$OUT/bench.log" 2> "$OUT/bench.err" || { echo bench failed; tail -5 "$OUT/bench.err"; }
tail -1 "$OUT/bench.log" | cut -c1-400
( time python bench.py --impl reference --gpus 1 --steps 3 --warmup 1 ) > "$OUT/ref.log" 2>&1; grep -h '^{' "$OUT/ref.log" | cut -c1-300; grep real "$OUT/ref.log"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k 'regex:lora_|adamw|reduce_splits|gather_rows' -c 4000 --csv --log-file "$OUT/launches.csv" \
  python bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline --aimd-steps 0 > "$OUT/ncu_launches.log" 2>&1
echo "ncu rc $?"; wc -l "$OUT/launches.csv"
