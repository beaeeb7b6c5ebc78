#!/bin/bash
# Functional runs of the bench variants on one GPU: the reference arm, and the
# episode-sharded multi-rank path with two ranks sharing GPU 0 over gloo.
mkdir -p gpurun_out
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
EPI_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_w2_cfg2.json 2> gpurun_out/bench_w2_cfg2.err
EPI_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --config cfg1 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_w2_cfg1.json 2> gpurun_out/bench_w2_cfg1.err
EPI_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 2 --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/bench_w2_cfg3.json 2> gpurun_out/bench_w2_cfg3.err
