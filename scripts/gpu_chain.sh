#!/bin/bash
# chain kernel: parity tests, then cfg3 / cfg5 10Mx1M bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_chain.py -q -x 2>&1 | tail -15 > gpurun_out/pytest_chain.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k "not 1000000000" 2>&1 | tail -15 > gpurun_out/pytest_scale.log
timeout 300 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 600 python bench.py --config cfg5 --cfg5-cands 1000000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_1M.json 2> gpurun_out/bench_cfg5_1M.err
timeout 1200 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
