#!/bin/bash
# Slot-list row mode (_lib_s) vs the current chain kernel (_lib): chain/scale
# parity on _lib_s, bench lines of both, ncu capture of the slot kernel.
O=gpurun_out/slot; mkdir -p $O
W='import faulthandler,sys,runpy; faulthandler.dump_traceback_later(int(sys.argv[1]), exit=True); sys.argv=["bench.py"]+sys.argv[2:]; runpy.run_path("bench.py", run_name="__main__")'
export EPI_LIB=$PWD/paper_0905_2203_b200/_lib_s/libepisodic_b200.so
timeout 400 python -m pytest tests/test_gpu_chain.py tests/test_gpu_scale.py tests/test_gpu_multi.py -m gpu -q --timeout 180 --timeout-method thread > $O/pytest_s.log 2>&1
for v in _lib_s _lib; do
  export EPI_LIB=$PWD/paper_0905_2203_b200/$v/libepisodic_b200.so
  timeout 130 python -u -c "$W" 120 --steps 5 --warmup 3 --no-cpu-baseline > $O/cfg5$v.json 2> $O/cfg5$v.err
  timeout 100 python -u -c "$W" 90 --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline > $O/cfg2$v.json 2> $O/cfg2$v.err
done
export EPI_LIB=$PWD/paper_0905_2203_b200/_lib_s/libepisodic_b200.so
timeout 400 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -c 1 -o $O/prof_slot_cfg5 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_slot.log 2>&1
