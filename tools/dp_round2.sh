#!/bin/bash
# usage: dp_round2.sh OUTDIR NGPU  (under gpurun --gpus NGPU)
OUT=$1; N=$2
mkdir -p "$OUT"
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"),
      (d.get("roofline") or {}).get("frac"), flush=True)
PY
}
two() { local name=$1; local envs=$2; shift 2; env $envs python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $N "$@" > "$OUT/$name.log" 2>&1; summ "$OUT/$name.log" $name; }
python -m pytest tests/test_gpu_executor.py -q -k data_parallel > "$OUT/dp_check.log" 2>&1; tail -1 "$OUT/dp_check.log"
two c2_dp X=0 --steps 20 --warmup 5 --aimd-steps 0
two c2_dp_static TLORA_DYN_SCHED=0 --steps 20 --warmup 5 --aimd-steps 0
two c2_dp_b X=0 --steps 20 --warmup 5 --aimd-steps 0
two c3_dp X=0 --config C3 --steps 4 --warmup 3 --aimd-steps 0
two c3_dp_sharded X=0 --config C3 --steps 4 --warmup 3 --aimd-steps 0 --dp-sharded-opt
