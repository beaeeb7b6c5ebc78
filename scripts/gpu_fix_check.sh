#!/bin/bash
# The prologue shuffle fix: GPU suite + smoke + bench lines on the in-tree
# build; the slot-list/rebuild-check variant (_lib_n) on the chain/scale
# tests and the cfg5/cfg3 cells.
O=gpurun_out/fix; mkdir -p $O
timeout 600 python -m pytest tests/ -q -m gpu --timeout 240 --timeout-method thread > $O/pytest_gpu.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 300 python bench.py > $O/r02_bench_default.json 2> $O/default.err
EPI_LIB=$PWD/paper_0905_2203_b200/_lib_n/libepisodic_b200.so timeout 300 python -m pytest tests/test_gpu_chain.py tests/test_gpu_scale.py tests/test_gpu_parity.py -q -m gpu --timeout 120 --timeout-method thread > $O/pytest_n.log 2>&1
EPI_LIB=$PWD/paper_0905_2203_b200/_lib_n/libepisodic_b200.so timeout 200 python bench.py --steps 10 --no-cpu-baseline > $O/cfg5_n.json 2> $O/cfg5_n.err
EPI_LIB=$PWD/paper_0905_2203_b200/_lib_n/libepisodic_b200.so timeout 200 python bench.py --config cfg3 --steps 20 --no-cpu-baseline > $O/cfg3_n.json 2> $O/cfg3_n.err
timeout 200 python bench.py --config cfg3 --steps 20 > $O/r02_bench_cfg3.json 2> $O/cfg3.err
