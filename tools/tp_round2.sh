#!/bin/bash
# TP evidence (under gpurun --gpus N): C++ TP step vs the Python driver, AIMD vs fixed N.
OUT=$1; N=$2
mkdir -p "$OUT"
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
c = d.get("config") or {}
tr = c.get("aimd_trajectory_n_ms") or []
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"),
      "N:", [t[0] for t in tr][:12], c.get("nano_batches"), flush=True)
PY
}
run() { local name=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $N --tp "$@" > "$OUT/$name.log" 2>&1; summ "$OUT/$name.log" $name; }
[ "$N" -ge 2 ] && TP_CONFIG=C2 TP_NANO=3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29612 tests/tp_exec_check.py > "$OUT/tp_exec_check.log" 2>&1; grep TP_EXEC "$OUT/tp_exec_check.log"
run cpp_aimd --steps 12 --warmup 3
run cpp_n2 --steps 8 --warmup 3 --nano-batches 2
run cpp_n3 --steps 8 --warmup 3 --nano-batches 3
run python_driver --steps 8 --warmup 3 --tp-driver python
run cpp_aimd_b --steps 12 --warmup 3
