#!/bin/bash
# Round-2 evidence at HEAD (1 GPU): launch list of the benched step, DRAM traffic of the 14
# fused GEMMs, ncu --set full of a deep fused GEMM (down fwd), the AdamW launches and the
# dB+dA launches of one step.  usage: profile_r2.sh OUTDIR COMMIT
OUT=$1; COMMIT=$2
mkdir -p "$OUT"
python tools/prof_step.py --warmup 2 --steps 1 > "$OUT/plain.log" 2>&1 || exit 1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --aimd-steps 0 > "$OUT/bench_plain.log" 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-cpu-baseline --aimd-steps 0 > "$OUT/ncu_launches.log" 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:lora_gemm2 --launch-skip 31 -c 14 --csv \
  --log-file "$OUT/traffic14.csv" python tools/prof_step.py --warmup 2 --steps 1 > "$OUT/ncu_traffic.log" 2>&1
python tools/traffic_from_ncu.py "$OUT/traffic14.csv" "$COMMIT" "$OUT/traffic.json" > "$OUT/traffic_summary.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lora_gemm2 -s 37 -c 1 \
  -o "$OUT/fwd_down" python tools/prof_step.py --warmup 2 --steps 1 > "$OUT/ncu_fwd_down.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:adamw -s 14 -c 7 \
  -o "$OUT/adamw" python tools/prof_step.py --warmup 2 --steps 1 > "$OUT/ncu_adamw.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lora_grad -s 14 -c 7 \
  -o "$OUT/grads" python tools/prof_step.py --warmup 2 --steps 1 > "$OUT/ncu_grads.log" 2>&1
ls -la "$OUT"
