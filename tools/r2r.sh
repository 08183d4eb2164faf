#!/bin/bash
OUT=$1; N=2
mkdir -p "$OUT"
summ() { python - "$1" "$2" <<'PY'
import json, sys
lines = [l for l in open(sys.argv[1]).read().splitlines() if l.startswith("{")]
d = json.loads(lines[-1]) if lines else {}
print(sys.argv[2], d.get("value"), d.get("ms_per_step"), (d.get("clocks") or {}).get("sm_mhz"),
      (d.get("roofline") or {}).get("frac"), flush=True)
PY
}
one() { local name=$1; shift; CUDA_VISIBLE_DEVICES=0 python bench.py "$@" > "$OUT/$name.log" 2>&1; summ "$OUT/$name.log" $name; }
tp() { local name=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) bench.py --gpus $N --tp "$@" > "$OUT/$name.log" 2>&1; summ "$OUT/$name.log" $name; }
one n1_a --steps 20 --warmup 5 --no-cpu-baseline
tp tp2_cpp_n2 --steps 8 --warmup 3 --nano-batches 2
tp tp2_py_n2 --steps 8 --warmup 3 --tp-driver python --nano 2 --aimd-steps 0
tp tp2_cpp_n3 --steps 8 --warmup 3 --nano-batches 3
tp tp2_py_n3 --steps 8 --warmup 3 --tp-driver python --nano 3 --aimd-steps 0
one n1_b --steps 20 --warmup 5 --no-cpu-baseline
