cd $GRAFT_REPO_ROOT
python scripts/python_overhead.py > gpurun_out/trace.txt 2>&1
EPI_TRACE=1 python - >> gpurun_out/trace.txt 2>&1 <<'PY'
import sys; sys.path.insert(0,'.')
import bench
from paper_0905_2203_b200 import Context, MODE_MINE
types, times, _ = bench.make_stream("cfg2")
ctx = Context(0); ctx.load_arrays(types, times, 26)
for i in range(8):
    print("---- iter", i, file=sys.stderr, flush=True)
    ctx.mine_raw(250, bench.BINS, 4, MODE_MINE)
PY
