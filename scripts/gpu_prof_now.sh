#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o gpurun_out/prof_now_cfg5 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_now.log 2>&1
