#!/bin/bash
# TP evidence after the timed-region fix (under gpurun --gpus N): C++ TP step with AIMD every
# step and with fixed N, the Python driver, interleaved twice.
OUT=$1; N=${2:-4}
mkdir -p "$OUT"
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
c = d.get("config") or {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"),
      c.get("nano_batches"), [x[0] for x in c.get("aimd_trajectory_n_ms", [])],
      (d.get("pipeline_monitor") or {}).get("eta_util"), flush=True)
PY
}
run() { local name=$1; local envs=$2; shift 2; env $envs python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $N "$@" > "$OUT/$name.log" 2>&1; summ "$OUT/$name.log" $name; }
for rep in 1 2; do
run cpp_aimd_$rep X=0 --tp --steps 10 --warmup 3
run cpp_n2_$rep X=0 --tp --steps 10 --warmup 3 --nano-batches 2
run cpp_n4_$rep X=0 --tp --steps 10 --warmup 3 --nano-batches 4
run py_$rep X=0 --tp --steps 10 --warmup 3 --tp-driver python
done
