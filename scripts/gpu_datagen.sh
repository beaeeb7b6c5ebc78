#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_datagen.py -q -x 2>&1 | tail -15 > gpurun_out/pytest_datagen.log
python - > gpurun_out/gen_timing.txt 2>&1 <<'PY'
import time, sys
sys.path.insert(0, ".")
import torch
from paper_0905_2203_b200 import Context, GenConfig, generate_arrays
ctx = Context(0)
for n in (10_000_000, 100_000_000, 1_000_000_000):
    cfg = GenConfig(64, n / 1280, 20, [], 5 + n)
    ctx.generate(cfg)
    t0 = time.perf_counter(); ctx.generate(cfg); torch.cuda.synchronize(); t1 = time.perf_counter()
    if n <= 100_000_000:
        h0 = time.perf_counter(); generate_arrays(cfg); h1 = time.perf_counter()
        host = f"host generate_arrays {h1-h0:.2f} s"
    else:
        host = ""
    print(f"n={n}: device generate+load {1e3*(t1-t0):.1f} ms {host}", flush=True)
PY
