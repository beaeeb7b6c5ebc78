import os, sys, time, ctypes as C
sys.path.insert(0, "/root/repo")
import numpy as np
import bench
from paper_0905_2203_b200 import Context, MODE_MINE, _native as N
types, times, _ = bench.make_stream("cfg2")
ctx = Context(0)
ctx.load_arrays(types, times, 26)
for _ in range(5): ctx.mine_raw(250, bench.BINS, 4, MODE_MINE)
cfg = ctx._mine_cfg[1]
ts, tc = [], []
for _ in range(50):
    t0 = time.perf_counter(); ctx.mine_raw(250, bench.BINS, 4, MODE_MINE); t1 = time.perf_counter()
    res = N.MineResultOut()
    t2 = time.perf_counter(); N.lib.epi_mine(ctx._h, C.byref(cfg), C.byref(res)); t3 = time.perf_counter()
    ts.append(t1 - t0); tc.append(t3 - t2)
print("mine_raw median %.1f us, raw ctypes call median %.1f us" % (np.median(ts) * 1e6, np.median(tc) * 1e6))
