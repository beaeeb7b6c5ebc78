#!/bin/bash
# Round-2 evidence: default bench line (with CPU baseline), reference arm,
# cfg2 with its reference arm (full mine()), launch list + full ncu capture
# of the default config's dominant kernel.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/nproc.txt
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
timeout 600 python bench.py --config cfg2 --steps 20 > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err
timeout 900 python bench.py --config cfg2 --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_cfg2_reference.json 2> gpurun_out/r02_bench_cfg2_reference.err
timeout 600 python bench.py --config cfg3 --steps 10 > gpurun_out/r02_bench_cfg3.json 2> gpurun_out/r02_bench_cfg3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_default.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o gpurun_out/r02_prof_chain_default -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_default.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o gpurun_out/r02_prof_chain_cfg3 -f python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_cfg3.log 2>&1
