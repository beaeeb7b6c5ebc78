#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "encoded_ingest" 2>&1 | tail -5 > gpurun_out/pytest_ingest.log
timeout 1500 python scripts/ingest_bench.py 10000000 100000000 1000000000 > gpurun_out/r02_ingest.jsonl 2> gpurun_out/r02_ingest.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 900 python bench.py --cfg5-events 1000000000 --cfg5-cands 1000 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_1B_1k.json 2> gpurun_out/bench_1B_1k.err
