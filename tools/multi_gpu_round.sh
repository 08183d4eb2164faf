# Multi-GPU measurements on one 4-GPU box (gpurun --gpus 4): DP weak scaling of C2 and C3,
# TP strong scaling of the C4 layer. One JSON line per run under gpurun_out/mg/.
mkdir -p gpurun_out/mg
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 400 $R --nproc-per-node 4 --master-port 29511 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/mg/c2_dp4.log 2>&1
timeout 400 $R --nproc-per-node 2 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/mg/c2_dp2.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/mg/c2_dp1.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29513 bench.py --gpus 4 --config C3 --steps 3 --warmup 3 > gpurun_out/mg/c3_dp4.log 2>&1
timeout 600 $R --nproc-per-node 2 --master-port 29516 bench.py --gpus 2 --config C3 --steps 3 --warmup 3 > gpurun_out/mg/c3_dp2.log 2>&1
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mg/c3_dp1.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29514 bench.py --gpus 4 --tp --config C4 --steps 5 --warmup 3 > gpurun_out/mg/c4_tp4.log 2>&1
timeout 600 $R --nproc-per-node 2 --master-port 29515 bench.py --gpus 2 --tp --config C4 --steps 5 --warmup 3 > gpurun_out/mg/c4_tp2.log 2>&1
for f in gpurun_out/mg/*.log; do echo "== $f"; grep '^{' $f | tail -1 | cut -c1-300; done
