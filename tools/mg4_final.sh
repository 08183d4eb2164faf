#!/bin/bash
# Final 4-GPU evidence (under gpurun --gpus 4): every multi-GPU test at 4 ranks, DP4 C2,
# TP4 C4 (C++ step and Python driver), NVLink counters of the fused GEMM + reduce-scatter
# at world 4 (single process under ncu).
OUT=$1; N=4
mkdir -p "$OUT"
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"),
      (d.get("pipeline_monitor") or {}).get("eta_util"), flush=True)
PY
}
run() { local name=$1; local envs=$2; shift 2; env $envs python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $N "$@" > "$OUT/$name.log" 2>&1; summ "$OUT/$name.log" $name; }
python -m pytest tests -q -m gpu -k "multi_gpu or data_parallel" > "$OUT/mg_tests.log" 2>&1; tail -1 "$OUT/mg_tests.log"
python tools/gemm_rs_nvlink.py --world 4 > "$OUT/gemm_rs_plain.log" 2>&1 && \
ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:lora_gemm2 --csv --log-file "$OUT/gemm_rs_tp4_nvlink.csv" \
    python tools/gemm_rs_nvlink.py --world 4 > "$OUT/gemm_rs_ncu.log" 2>&1
cat "$OUT/gemm_rs_plain.log"
run c2_dp4 X=0 --steps 20 --warmup 5 --aimd-steps 0
run c4_tp4_cpp X=0 --tp --steps 8 --warmup 3
run c4_tp4_cpp_n2 X=0 --tp --steps 8 --warmup 3 --nano-batches 2
run c4_tp4_py X=0 --tp --steps 8 --warmup 3 --tp-driver python
