#!/bin/bash
# A/B of two in-tree library builds on the bench configs (EPI_LIB selects one)
mkdir -p gpurun_out
for v in _lib _lib_b3; do
  EPI_LIB=$PWD/paper_0905_2203_b200/$v/libepisodic_b200.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_default$v.json 2>&1
  EPI_LIB=$PWD/paper_0905_2203_b200/$v/libepisodic_b200.so timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_cfg3$v.json 2>&1
done
