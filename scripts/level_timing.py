"""Per-level host wall time vs device time of cfg2 mining (diagnostics)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_0905_2203_b200 import Context, MODE_MINE
types, times, _ = bench.make_stream("cfg2")
ctx = Context(0)
ctx.load_arrays(types, times, 26)
for it in range(5):
    t0 = time.perf_counter()
    cands, offs, ms, csr, counts, st = ctx.mine_raw(250, bench.BINS, 4, MODE_MINE)
    t1 = time.perf_counter()
    if it >= 3:
        print("wall %.3f ms; level host ms %s; device total %.3f ms (map %.3f walk %.3f p1 %.3f p2 %.3f); launches %d"
              % ((t1 - t0) * 1e3, [round(x, 3) for x in ms], st["total_ms"], st["map_ms"], st["concat_ms"],
                 st["pass1_ms"], st["pass2_ms"], st["kernel_launches"]))
