#!/bin/bash
# Closing run of the committed build: GPU suite, smoke, default + cfg3 + cfg2
# bench lines, launch list and ncu capture of the default cell's chain kernel.
O=gpurun_out/closing; mkdir -p $O
timeout 600 python -m pytest tests/ -q -m gpu --timeout 240 --timeout-method thread > $O/pytest_gpu.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 300 python bench.py > $O/r02_bench_default.json 2> $O/default.err
timeout 200 python bench.py --config cfg3 --steps 20 > $O/r02_bench_cfg3.json 2> $O/cfg3.err
timeout 200 python bench.py --config cfg2 --steps 50 > $O/r02_bench_cfg2.json 2> $O/cfg2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_default.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o $O/r02_prof_chain_default -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_default.log 2>&1
