#!/bin/bash
# GPU suite file by file; a hung test is dumped and killed (thread method).
O=gpurun_out/suite; mkdir -p $O
VERBOSE=1 timeout 150 tests/cpp/_build/adaptor_test > $O/adaptor.log 2>&1; echo "rc=$?" >> $O/adaptor.log
for f in test_gpu_chain test_gpu_parity test_gpu_multi test_gpu_shard test_gpu_scale test_gpu_tracking test_gpu_datagen; do
  timeout 600 python -m pytest tests/$f.py -m gpu -v --timeout 180 --timeout-method thread --durations 15 > $O/$f.log 2>&1
done
