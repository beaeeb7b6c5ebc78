#!/bin/bash
# ncu captures of the chain map kernel (cfg3 and the cfg5 10M x 1M cell)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o gpurun_out/prof_chain_cfg3 -f python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_chain_cfg3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o gpurun_out/prof_chain_cfg5 -f python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_chain_cfg5.log 2>&1
