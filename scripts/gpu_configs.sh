#!/bin/bash
# Bench lines of the counting configs beyond cfg1-3 (cfg4 MEA-shaped, cfg5
# sweep cells) on one GPU; outputs in gpurun_out/.
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
for cell in "1000000 1000" "10000000 10000" "10000000 100000" "100000000 1000" "100000000 10000"; do
  set -- $cell
  timeout 900 python bench.py --config cfg5 --cfg5-events $1 --cfg5-cands $2 --steps 3 --warmup 3 --cpu-seconds 3 \
    > gpurun_out/bench_cfg5_${1}_${2}.json 2> gpurun_out/bench_cfg5_${1}_${2}.err
done
