# 4-GPU re-check: multi-GPU parity tests and the DP / TP bench lines (gpurun --gpus 4)
mkdir -p gpurun_out/r1d4b
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -q -k "tp or dp or comm" > gpurun_out/r1d4b/pytest_mg.log 2>&1; echo "rc=$?" >> gpurun_out/r1d4b/pytest_mg.log
env | grep NCCL > gpurun_out/r1d4b/nccl_env.txt
timeout 400 $R --nproc-per-node 4 --master-port 29512 bench.py --gpus 4 > gpurun_out/r1d4b/c2_dp4.json 2> gpurun_out/r1d4b/c2_dp4.err
tail -3 gpurun_out/r1d4b/pytest_mg.log; cat gpurun_out/r1d4b/nccl_env.txt; head -c 300 gpurun_out/r1d4b/c2_dp4.json
