#!/bin/bash
# Bench lines of the committed build (default cell with its CPU baseline, cfg3, cfg2).
O=gpurun_out/final2; mkdir -p $O
timeout 400 python bench.py > $O/r02_bench_default.json 2> $O/default.err
timeout 300 python bench.py --config cfg3 --steps 20 > $O/r02_bench_cfg3.json 2> $O/cfg3.err
timeout 300 python bench.py --config cfg2 --steps 50 > $O/r02_bench_cfg2.json 2> $O/cfg2.err
timeout 600 python bench.py --config cfg4 --steps 5 > $O/r02_bench_cfg4.json 2> $O/cfg4.err
