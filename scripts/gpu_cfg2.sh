#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg2 or pass1 or mine" 2>&1 | tail -3 > gpurun_out/pytest_cfg2.log
python scripts/level_timing.py > gpurun_out/level_timing.txt 2>&1
timeout 300 python bench.py --config cfg2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
