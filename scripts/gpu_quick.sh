#!/bin/bash
# Quick GPU round-trip: the GPU test suite (or a subset via TESTS), then
# the cfg2 bench line and a two-rank functional run.
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests/} -q -m gpu -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 300 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
EPI_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_w2_cfg2.json 2> gpurun_out/bench_w2_cfg2.err
python scripts/level_timing.py > gpurun_out/level_timing.txt 2>&1
