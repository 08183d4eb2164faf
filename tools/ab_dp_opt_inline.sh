# A/B of TLORA_DP_OPT_INLINE at DP2 (per-projection AdamW on the comm stream vs at step end)
mkdir -p gpurun_out/abdp
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
p=29600
for rep in 1 2 3; do
for inl in 0 1; do
p=$((p+1))
TLORA_DP_OPT_INLINE=$inl timeout 300 $R --master-port $p bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/abdp/inl${inl}_$rep.json 2>gpurun_out/abdp/inl${inl}_$rep.err
python -c "import json; d=json.loads(open('gpurun_out/abdp/inl${inl}_$rep.json').read().strip().splitlines()[-1]); print('inline $inl rep $rep', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'])"
done; done
