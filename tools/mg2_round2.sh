#!/bin/bash
# 2-GPU evidence (under gpurun --gpus 2): executor DP check, NVLink counter probe, TP2 C4
# (fused GEMM + reduce-scatter vs NCCL), C2 DP2 dynamic vs static tile scheduler.
OUT=$1; N=2
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
python tools/nvlink_probe.py > "$OUT/nvlink_probe.log" 2>&1
python -m pytest tests/test_gpu_executor.py -q -s -k data_parallel > "$OUT/dp_check.log" 2>&1; tail -1 "$OUT/dp_check.log"
run c4_tp2 X=0 --tp --steps 6 --warmup 3
run c4_tp2_nccl X=0 --tp --steps 6 --warmup 3 --fused-rs none
run c2_dp_dyn X=0 --steps 20 --warmup 5 --aimd-steps 0
run c2_dp_static TLORA_DYN_SCHED=0 --steps 20 --warmup 5 --aimd-steps 0
run c2_dp_dyn_b X=0 --steps 20 --warmup 5 --aimd-steps 0
run c2_dp_static_b TLORA_DYN_SCHED=0 --steps 20 --warmup 5 --aimd-steps 0
