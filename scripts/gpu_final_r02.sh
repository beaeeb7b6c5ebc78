#!/bin/bash
# Round-2 final evidence: GPU suite, smoke, every bench line, launch list and
# full ncu capture of the default config's dominant kernel.
mkdir -p gpurun_out/final
O=gpurun_out/final
nproc > $O/host.txt; grep -m1 "model name" /proc/cpuinfo >> $O/host.txt; nvidia-smi --query-gpu=name,clocks.max.sm --format=csv >> $O/host.txt
timeout 1800 python -m pytest tests/ -q -m gpu 2>&1 | tail -6 > $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/r02_bench_default.json 2> $O/default.err
timeout 900 python bench.py --impl reference > $O/r02_bench_reference.json 2> $O/reference.err
timeout 600 python bench.py --config cfg3 --steps 20 > $O/r02_bench_cfg3.json 2> $O/cfg3.err
timeout 600 python bench.py --config cfg2 --steps 50 > $O/r02_bench_cfg2.json 2> $O/cfg2.err
timeout 900 python bench.py --config cfg2 --impl reference --steps 3 --warmup 1 > $O/r02_bench_cfg2_reference.json 2> $O/cfg2r.err
timeout 900 python bench.py --config cfg4 --steps 5 > $O/r02_bench_cfg4.json 2> $O/cfg4.err
timeout 600 python bench.py --config cfg1 --steps 20 > $O/r02_bench_cfg1.json 2> $O/cfg1.err
for cell in "1000000 1000" "10000000 10000" "10000000 100000" "100000000 10000" "1000000000 1000" "1000000000 10000"; do
  set -- $cell
  timeout 900 python bench.py --cfg5-events $1 --cfg5-cands $2 --steps 5 > $O/r02_bench_cfg5_$1_$2.json 2> $O/cfg5_$1_$2.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_default.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o $O/r02_prof_chain_default -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_default.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o $O/r02_prof_chain_cfg3 -f python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_cfg3.log 2>&1
