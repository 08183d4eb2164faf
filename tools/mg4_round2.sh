#!/bin/bash
# 4-GPU evidence (under gpurun --gpus 4): executor DP4 (C2, C3), the multi-GPU tests at 4
# ranks, TP4 C4 layer with the fused GEMM + reduce-scatter (NVLink counters in the line),
# static vs dynamic tile scheduler.  usage: mg4_round2.sh OUTDIR
OUT=$1; N=4
mkdir -p "$OUT"
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
nv = d.get("nvlink") or {}
tx = sum(v["tx_bytes_per_step"] for v in (nv.get("per_gpu") or {}).values()) if nv else None
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"),
      "nvlink_tx_GB_per_step=%s" % (None if tx is None else round(tx / 1e9, 3)), flush=True)
PY
}
run() { local name=$1; local envs=$2; shift 2; env $envs python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $N "$@" > "$OUT/$name.log" 2>&1; summ "$OUT/$name.log" $name; }
python -m pytest tests -q -m gpu -k "multi_gpu or data_parallel" > "$OUT/mg_tests.log" 2>&1; tail -1 "$OUT/mg_tests.log"
run c2_dp4 X=0 --steps 20 --warmup 5 --aimd-steps 0
run c3_dp4 X=0 --config C3 --steps 4 --warmup 3 --aimd-steps 0
run c4_tp4 X=0 --tp --steps 6 --warmup 3
run c4_tp4_dyn TLORA_DYN_SCHED=1 --tp --steps 6 --warmup 3
run c4_tp4_nccl X=0 --tp --steps 6 --warmup 3 --fused-rs none
