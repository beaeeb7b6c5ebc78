#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_cpp_adaptor.py tests/test_gpu_tracking.py -q -x 2>&1 | tail -15 > gpurun_out/pytest_multi.log
python - > gpurun_out/multi_nccl.txt 2>&1 <<'PY'
import numpy as np
from paper_0905_2203_b200 import Context
m = Context(devices=[0])
print("world", m.world, "nccl", m.uses_nccl)
m.close()
PY
