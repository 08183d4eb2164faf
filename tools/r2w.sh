#!/bin/bash
OUT=$1; N=2
mkdir -p "$OUT"
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"), [t[1] for t in (d.get("config") or {}).get("aimd_trajectory_n_ms", [])], flush=True)
PY
}
tp() { local name=$1; local envs=$2; shift 2; env $envs python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $N --tp "$@" > "$OUT/$name.log" 2>&1; summ "$OUT/$name.log" $name; }
tp cpp_traced "TLORA_DYN_SCHED=1 TLORA_TP_TRACE_ALL=1" --steps 8 --warmup 3 --nano-batches 2
tp cpp "TLORA_DYN_SCHED=1" --steps 8 --warmup 3 --nano-batches 2
tp cpp_sync "TLORA_DYN_SCHED=1 TLORA_TP_SYNC=1" --steps 8 --warmup 3 --nano-batches 2
tp py "TLORA_DYN_SCHED=1" --steps 8 --warmup 3 --tp-driver python --nano 2 --aimd-steps 0
