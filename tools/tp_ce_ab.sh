# TP: copy-engine all-gather + push reduce-scatter (default) vs NCCL (TLORA_TP_CE_AG=0); parity first.
mkdir -p gpurun_out/tpce2
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
TP_FUSED_RS=1 timeout 300 $R --nproc-per-node 2 --master-port 29601 tests/tp_check.py > gpurun_out/tpce2/check2.log 2>&1; echo rc=$? >> gpurun_out/tpce2/check2.log
TP_FUSED_RS=1 timeout 300 $R --nproc-per-node 4 --master-port 29602 tests/tp_check.py > gpurun_out/tpce2/check4.log 2>&1; echo rc=$? >> gpurun_out/tpce2/check4.log
timeout 300 $R --nproc-per-node 4 --master-port 29603 tests/tp_check.py > gpurun_out/tpce2/check4_nofused.log 2>&1; echo rc=$? >> gpurun_out/tpce2/check4_nofused.log
for r in 1 2; do
timeout 400 $R --nproc-per-node 4 --master-port 2961$r bench.py --gpus 4 --tp --config C4 --steps 5 --warmup 3 > gpurun_out/tpce2/tp4_ce_$r.log 2>&1
TLORA_TP_CE_AG=0 timeout 400 $R --nproc-per-node 4 --master-port 2962$r bench.py --gpus 4 --tp --config C4 --steps 5 --warmup 3 > gpurun_out/tpce2/tp4_nccl_$r.log 2>&1
done
timeout 400 $R --nproc-per-node 2 --master-port 29631 bench.py --gpus 2 --tp --config C4 --steps 5 --warmup 3 > gpurun_out/tpce2/tp2_ce.log 2>&1
TLORA_TP_CE_AG=0 timeout 400 $R --nproc-per-node 2 --master-port 29632 bench.py --gpus 2 --tp --config C4 --steps 5 --warmup 3 > gpurun_out/tpce2/tp2_nccl.log 2>&1
