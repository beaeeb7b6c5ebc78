#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_scale.py -q -x -k "not 1000000000" 2>&1 | tail -15 > gpurun_out/pytest_chain.log
timeout 300 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_1M.json 2> gpurun_out/bench_cfg5_1M.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o gpurun_out/prof_chain_cfg5 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_chain_cfg5.log 2>&1
