#!/bin/bash
# Chain kernel: masked-chain validation (_lib) vs automaton validation
# (_lib_aut): chain parity tests on the new build, A/B bench lines, ncu
# source-level capture of the default cell.
O=gpurun_out/vab; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_scale.py -q -m gpu -x 2>&1 | tail -8 > $O/pytest_chain.log
for v in _lib _lib_aut; do
  EPI_LIB=$PWD/paper_0905_2203_b200/$v/libepisodic_b200.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/default$v.json 2>$O/default$v.err
  EPI_LIB=$PWD/paper_0905_2203_b200/$v/libepisodic_b200.so timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline > $O/cfg3$v.json 2>$O/cfg3$v.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o $O/prof_default -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_default.log 2>&1
