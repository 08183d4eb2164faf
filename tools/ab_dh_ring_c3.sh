# A/B of the backward dH ring depth on C3 (32 Llama-3-8B layers), interleaved, one GPU
mkdir -p gpurun_out/abc3
for rep in 1 2; do
for ring in 4 8; do
TLORA_DH_RING=$ring timeout 400 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/abc3/ring${ring}_$rep.json 2>gpurun_out/abc3/ring${ring}_$rep.err
python -c "import json; d=json.load(open('gpurun_out/abc3/ring${ring}_$rep.json')); print('ring $ring rep $rep', d['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
