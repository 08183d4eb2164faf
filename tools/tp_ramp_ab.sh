#!/bin/bash
# Ramped nano-batch sizes for the C++ TP step (TLORA_TP_RAMP=g) vs uniform, interleaved.
OUT=$1; N=${2:-4}
mkdir -p "$OUT"
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
pm = d.get("pipeline_monitor") or {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"),
      pm.get("eta_util"), pm.get("delta_stall_s"), flush=True)
PY
}
run() { local name=$1; local envs=$2; shift 2; env $envs python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $N "$@" > "$OUT/$name.log" 2>&1; summ "$OUT/$name.log" $name; }
for rep in 1 2; do
run n2_$rep X=0 --tp --steps 10 --warmup 3 --nano-batches 2
run n3g18_$rep TLORA_TP_RAMP=1.8 --tp --steps 10 --warmup 3 --nano-batches 3
run n4g18_$rep TLORA_TP_RAMP=1.8 --tp --steps 10 --warmup 3 --nano-batches 4
run n5g18_$rep TLORA_TP_RAMP=1.8 --tp --steps 10 --warmup 3 --nano-batches 5
run n4g25_$rep TLORA_TP_RAMP=2.5 --tp --steps 10 --warmup 3 --nano-batches 4
run n3g25_$rep TLORA_TP_RAMP=2.5 --tp --steps 10 --warmup 3 --nano-batches 3
done
