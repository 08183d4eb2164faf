mkdir -p gpurun_out/r1c
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1c/bench_plain.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r1c/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1c/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lora_gemm2 -s 9 -c 1 -o gpurun_out/r1c/fwd_gate_chain python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline > gpurun_out/r1c/ncu_gate.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather_rows -c 1 -o gpurun_out/r1c/gather python bench.py --steps 1 --warmup 3 --no-graph --shuffle --no-cpu-baseline > gpurun_out/r1c/ncu_gather.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lora_grad -s 4 -c 1 -o gpurun_out/r1c/grad python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline > gpurun_out/r1c/ncu_grad.log 2>&1
ls -la gpurun_out/r1c
