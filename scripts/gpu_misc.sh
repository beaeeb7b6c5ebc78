#!/bin/bash
mkdir -p gpurun_out
python scripts/level_timing.py > gpurun_out/level_timing.txt 2>&1
EPI_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_w2_default.json 2> gpurun_out/bench_w2_default.err
EPI_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --config cfg2 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_w2_cfg2.json 2> gpurun_out/bench_w2_cfg2.err
