#!/bin/bash
# Where do the C++ TP step's back-to-back milliseconds go? (under gpurun --gpus N)
OUT=$1; N=${2:-4}
mkdir -p "$OUT"
run() { local name=$1; local envs=$2; shift 2; env $envs python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $N "$@" > "$OUT/$name.log" 2>&1; grep -h "rank 0\]" "$OUT/$name.log" | tail -12; grep -o '"ms_per_step": [0-9.]*' "$OUT/$name.log"; }
run sync "TLORA_TP_SYNC=1 TLORA_TP_DEBUG=1 TLORA_BENCH_STEP_EVENTS=1" --tp --steps 8 --warmup 3 --nano-batches 2
run lazy "TLORA_TP_DEBUG=1 TLORA_BENCH_STEP_EVENTS=1" --tp --steps 8 --warmup 3 --nano-batches 2
run py "TLORA_BENCH_STEP_EVENTS=1" --tp --steps 8 --warmup 3 --nano-batches 2 --tp-driver python
run lazy_n4 "TLORA_TP_DEBUG=1 TLORA_BENCH_STEP_EVENTS=1" --tp --steps 8 --warmup 3 --nano-batches 4
run py_fixed2 "TLORA_BENCH_STEP_EVENTS=1" --tp --steps 8 --warmup 3 --nano-batches 2 --aimd-steps 0 --tp-driver python
