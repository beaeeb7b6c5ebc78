#!/bin/bash
# Diagnose slow/hanging GPU tests and bench: per-step logs streamed to files.
O=gpurun_out/diag; mkdir -p $O
nproc > $O/host.txt; nvidia-smi >> $O/host.txt 2>&1
EPI_LIB=$PWD/paper_0905_2203_b200/_lib_aut/libepisodic_b200.so timeout 300 python -u bench.py --steps 5 --no-cpu-baseline > $O/bench_old.json 2> $O/bench_old.err
timeout 300 python -u bench.py --steps 5 --no-cpu-baseline > $O/bench_new.json 2> $O/bench_new.err
timeout 300 python -u bench.py --config cfg3 --steps 5 --no-cpu-baseline > $O/cfg3_new.json 2> $O/cfg3_new.err
timeout 1200 python -m pytest tests/ -m gpu -v -p pytest_timeout --timeout 240 --durations 40 > $O/pytest.log 2>&1
