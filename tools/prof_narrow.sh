#!/bin/bash
# ncu --set full of the narrow C2 launches (fwd k + shrink v, dX k + dH q) next to fwd q.
OUT=$1
mkdir -p "$OUT"
python tools/prof_step.py --warmup 2 --steps 1 > "$OUT/plain.log" 2>&1 || exit 1
for s in 31 32 43; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:lora_gemm2 -s $s -c 1 \
    -o "$OUT/gemm_s$s" python tools/prof_step.py --warmup 2 --steps 1 > "$OUT/ncu_s$s.log" 2>&1
done
ls -la "$OUT"
