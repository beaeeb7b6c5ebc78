#!/bin/bash
# Round-2 baseline: GPU tests, cfg3 / cfg5 10Mx1M bench lines, cfg3 map-kernel ncu.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 600 python bench.py --config cfg5 --cfg5-cands 1000000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_1M.json 2> gpurun_out/bench_cfg5_1M.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:machines_kernel -s 2 -c 1 -o gpurun_out/prof_cfg3 -f python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cfg3.log 2>&1
