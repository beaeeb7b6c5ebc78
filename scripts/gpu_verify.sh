#!/bin/bash
# Re-entry check of HEAD: GPU suite, smoke, default bench line, cfg3 line.
O=gpurun_out/verify; mkdir -p $O
timeout 1500 python -m pytest tests/ -q -m gpu 2>&1 | tail -15 > $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 600 python bench.py --steps 10 > $O/bench_default.json 2> $O/default.err
timeout 600 python bench.py --config cfg3 --steps 20 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/cfg3.err
timeout 600 python bench.py --config cfg2 --steps 20 --no-cpu-baseline > $O/bench_cfg2.json 2> $O/cfg2.err
