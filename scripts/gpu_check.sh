#!/bin/bash
# One GPU round-trip: parity tests, the three single-GPU bench configs, a
# launch list and full ncu captures of the dominant kernels. Outputs land in
# gpurun_out/ (merged back by gpurun).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 300 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 300 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
if [ "${NCU:-1}" = 1 ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:^bound_kernel -s 1 -c 1 -o gpurun_out/prof_bound -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bound.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:machines_kernel -s 3 -c 1 -o gpurun_out/prof_cfg2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cfg2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:machines_kernel -s 2 -c 1 -o gpurun_out/prof_cfg3 -f python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cfg3.log 2>&1
fi
