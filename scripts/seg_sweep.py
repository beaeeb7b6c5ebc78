"""Map-kernel time vs forced segment count (planner calibration)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_0905_2203_b200 import Context
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
types, times, a = bench.make_stream(cfg)
ctx = Context(0)
ctx.load_arrays(types, times, a)
csr = bench.count_candidates_csr(cfg)
for P in [None] + [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "8,11,15,18,22,26,29,37,44,59,74,89,118").split(",")]:
    if P is None:
        os.environ.pop("EPI_FORCE_SEGMENTS", None)
    else:
        os.environ["EPI_FORCE_SEGMENTS"] = str(P)
    best = 1e9
    for _ in range(4):
        ctx.count_csr(csr)
        st = ctx.last_stats
        best = min(best, st["map_ms"])
    print(f"P={st['segments']} forced={P} map_ms={best:.3f} concat_ms={st['concat_ms']:.3f} patches={st['patches']}", flush=True)
