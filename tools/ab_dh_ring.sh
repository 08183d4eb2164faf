# A/B of the backward dH ring depth (TLORA_DH_RING), interleaved, one GPU
mkdir -p gpurun_out/ab
for rep in 1 2 3; do
for ring in 4 8; do
TLORA_DH_RING=$ring timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab/ring${ring}_$rep.json 2>gpurun_out/ab/ring${ring}_$rep.err
python -c "import json; d=json.load(open('gpurun_out/ab/ring${ring}_$rep.json')); print('ring $ring rep $rep', d['ms_per_step'], d['clocks']['sm_mhz'], d['e2e']['value'])"
done; done
TLORA_DH_RING=8 timeout 600 python -m pytest tests -m gpu -q -x -k "chain or side or runner or layer_set" 2>&1 | tail -2
