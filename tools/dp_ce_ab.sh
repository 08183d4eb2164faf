# DP: copy-engine push all-reduce (TLORA_DP_CE=1) vs NCCL (default); correctness first.
mkdir -p gpurun_out/dpce
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $R --nproc-per-node 2 --master-port 29701 tests/dp_check.py > gpurun_out/dpce/check2.log 2>&1; echo rc=$? >> gpurun_out/dpce/check2.log
timeout 300 $R --nproc-per-node 4 --master-port 29702 tests/dp_check.py > gpurun_out/dpce/check4.log 2>&1; echo rc=$? >> gpurun_out/dpce/check4.log
for r in 1 2; do
TLORA_DP_CE=1 timeout 400 $R --nproc-per-node 4 --master-port 2971$r bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/dpce/dp4_ce_$r.log 2>&1
timeout 400 $R --nproc-per-node 4 --master-port 2972$r bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/dpce/dp4_nccl_$r.log 2>&1
done
TLORA_DP_CE=1 timeout 400 $R --nproc-per-node 2 --master-port 29731 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/dpce/dp2_ce.log 2>&1
timeout 400 $R --nproc-per-node 2 --master-port 29732 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/dpce/dp2_nccl.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/dpce/dp1.log 2>&1
