# A/B of the fused GEMM's dynamic tile scheduler (opt-in TLORA_DYN_SCHED=1) against the
# default static round-robin schedule, on one box, interleaved.
mkdir -p gpurun_out/dyn2
for r in 1 2 3 4; do
  TLORA_DYN_SCHED=1 timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/dyn2/dyn_$r.log 2>&1
  timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/dyn2/static_$r.log 2>&1
done
TLORA_DYN_SCHED=1 timeout 600 python bench.py --no-cpu-baseline --config C3 --steps 3 > gpurun_out/dyn2/c3_dyn.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --config C3 --steps 3 > gpurun_out/dyn2/c3_static.log 2>&1
