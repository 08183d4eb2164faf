#!/bin/bash
OUT=$1; N=2
mkdir -p "$OUT"
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"), flush=True)
PY
}
tp() { local name=$1; local envs=$2; shift 2; env $envs python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $N --tp "$@" > "$OUT/$name.log" 2>&1; summ "$OUT/$name.log" $name; }
tp cpp "TLORA_DYN_SCHED=1" --steps 8 --warmup 3 --nano-batches 2
tp cpp_memop_off "TLORA_DYN_SCHED=1 TLORA_TP_MEMOP_MAIN=0" --steps 8 --warmup 3 --nano-batches 2
tp cpp_b "TLORA_DYN_SCHED=1" --steps 8 --warmup 3 --nano-batches 2
tp py "TLORA_DYN_SCHED=1" --steps 8 --warmup 3 --tp-driver python --nano 2 --aimd-steps 0
tp cpp_memop_off_b "TLORA_DYN_SCHED=1 TLORA_TP_MEMOP_MAIN=0" --steps 8 --warmup 3 --nano-batches 2

