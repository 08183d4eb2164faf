#!/bin/bash
# DP efficiency diagnosis on C3 (run under gpurun --gpus 2): single-GPU graph vs eager, DP2
# variants.  usage: dp_diag.sh OUTDIR LAYERS
OUT=$1; L=$2
mkdir -p "$OUT"
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"),
      (d.get("roofline") or {}).get("frac"), flush=True)
PY
}
one() { local name=$1; shift; CUDA_VISIBLE_DEVICES=0 python bench.py --config C3 --layers $L --steps 6 --warmup 3 --aimd-steps 0 --no-cpu-baseline "$@" > "$OUT/$name.log" 2>&1; summ "$OUT/$name.log" $name; }
two() { local name=$1; local envs=$2; shift 2; env $envs python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus 2 --config C3 --layers $L --steps 6 --warmup 3 --aimd-steps 0 "$@" > "$OUT/$name.log" 2>&1; summ "$OUT/$name.log" $name; }
one n1_graph
one n1_eager --no-graph
two dp2 X=0
two dp2_dyn TLORA_DYN_SCHED=1
two dp2_nch4 NCCL_MAX_NCHANNELS=4
two dp2_sharded X=0 --dp-sharded-opt
