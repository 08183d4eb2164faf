#!/bin/bash
# DP evidence (run under gpurun --gpus N): executor DP check, C2 / C3 DP bench with the
# gradient all-reduce vs the sharded optimizer.  usage: dp_round.sh OUTDIR NGPU
OUT=$1; N=$2
mkdir -p "$OUT"
python -m pytest tests/test_gpu_executor.py -q -s -k data_parallel > "$OUT/dp_check.log" 2>&1
run() {  # name, bench args...
  local name=$1; shift
  python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 500)) bench.py --gpus "$N" "$@" > "$OUT/$name.log" 2>&1
  python - "$OUT/$name.log" "$name" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"), flush=True)
PY
}
run c2_ar --steps 20 --warmup 5 --aimd-steps 0
run c2_sharded --steps 20 --warmup 5 --aimd-steps 0 --dp-sharded-opt
run c2_ar_b --steps 20 --warmup 5 --aimd-steps 0
run c2_sharded_b --steps 20 --warmup 5 --aimd-steps 0 --dp-sharded-opt
run c3_ar --config C3 --steps 4 --warmup 3 --aimd-steps 0
run c3_sharded --config C3 --steps 4 --warmup 3 --aimd-steps 0 --dp-sharded-opt
