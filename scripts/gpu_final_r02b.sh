#!/bin/bash
# Round-2 closing evidence on the committed build: GPU suite, smoke, bench
# lines (default + reference arm, cfg3, cfg2 + reference, 1B x 1k), launch
# list and one ncu --set full capture of the default cell's chain kernel.
O=gpurun_out/final; mkdir -p $O
nproc > $O/host.txt; grep -m1 "model name" /proc/cpuinfo >> $O/host.txt
timeout 900 python -m pytest tests/ -q -m gpu --timeout 300 --timeout-method thread > $O/pytest_gpu.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 400 python bench.py > $O/r02_bench_default.json 2> $O/default.err
timeout 400 python bench.py --impl reference > $O/r02_bench_reference.json 2> $O/reference.err
timeout 300 python bench.py --config cfg3 --steps 20 > $O/r02_bench_cfg3.json 2> $O/cfg3.err
timeout 300 python bench.py --config cfg2 --steps 50 > $O/r02_bench_cfg2.json 2> $O/cfg2.err
timeout 400 python bench.py --config cfg2 --impl reference --steps 3 --warmup 1 > $O/r02_bench_cfg2_reference.json 2> $O/cfg2r.err
timeout 400 python bench.py --cfg5-events 1000000000 --cfg5-cands 1000 --steps 5 --no-cpu-baseline > $O/r02_bench_cfg5_1B_1k.json 2> $O/cfg5_1b.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_default.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o $O/r02_prof_chain_default -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_default.log 2>&1
