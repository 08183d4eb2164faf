#!/bin/bash
# A/B of the C++ TP step's synchronisation variants at TP=N (under gpurun --gpus N):
# back-to-back timed steps vs the library's own per-step event time.
OUT=$1; N=${2:-4}
mkdir -p "$OUT"
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
tr = [x[1] for x in (d.get("config") or {}).get("aimd_trajectory_n_ms", []) if x[1] and x[1] > 0]
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"),
      "lib_ms", tr[:4], "traced", (d.get("pipeline_monitor") or {}).get("t_iter_event_s"), flush=True)
PY
}
run() { local name=$1; local envs=$2; shift 2; env $envs python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $N "$@" > "$OUT/$name.log" 2>&1; summ "$OUT/$name.log" $name; }
for rep in 1 2; do
run memop_$rep X=0 --tp --steps 8 --warmup 3 --nano-batches 2
run kernel_$rep TLORA_TP_WAIT=kernel --tp --steps 8 --warmup 3 --nano-batches 2
run conn32_$rep CUDA_DEVICE_MAX_CONNECTIONS=32 --tp --steps 8 --warmup 3 --nano-batches 2
run sync_$rep TLORA_TP_SYNC=1 --tp --steps 8 --warmup 3 --nano-batches 2
run nccl_$rep TLORA_TP_CE_AG=0 --tp --steps 8 --warmup 3 --nano-batches 2 --fused-rs none
run py_$rep X=0 --tp --steps 8 --warmup 3 --nano-batches 2 --tp-driver python
done
run kernel_aimd TLORA_TP_WAIT=kernel --tp --steps 8 --warmup 3
run kernel_memmain0 "TLORA_TP_WAIT=kernel TLORA_TP_MEMOP_MAIN=0" --tp --steps 8 --warmup 3 --nano-batches 2
