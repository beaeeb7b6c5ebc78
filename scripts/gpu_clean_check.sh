#!/bin/bash
# The clean in-tree build (make from the committed sources): GPU suite, smoke, default bench line.
O=gpurun_out/clean; mkdir -p $O
timeout 600 python -m pytest tests/ -q -m gpu -x > $O/pytest_gpu.log 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 300 python bench.py > $O/r02_bench_default.json 2> $O/default.err
