#!/bin/bash
# 2-GPU: NVLink counters of the fused GEMM + reduce-scatter (single process, ncu), TP2 C4.
OUT=$1; N=2
mkdir -p "$OUT"
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"), flush=True)
PY
}
run() { local name=$1; local envs=$2; shift 2; env $envs python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $N "$@" > "$OUT/$name.log" 2>&1; summ "$OUT/$name.log" $name; }
python tools/gemm_rs_nvlink.py --world 2 > "$OUT/gemm_rs_plain.log" 2>&1 && \
ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:lora_gemm2 --csv --log-file "$OUT/gemm_rs_tp2_nvlink.csv" \
    python tools/gemm_rs_nvlink.py --world 2 > "$OUT/gemm_rs_ncu.log" 2>&1
cat "$OUT/gemm_rs_plain.log"
run c4_tp2 X=0 --tp --steps 6 --warmup 3
run c4_tp2_nccl X=0 --tp --steps 6 --warmup 3 --fused-rs none
run c4_tp2_static TLORA_DYN_SCHED=0 --tp --steps 6 --warmup 3
