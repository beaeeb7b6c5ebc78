"""Device parallel local tracking (epi_count_tracking) vs the bit-sliced
counter on the same batches: wall time per call and equality of counts."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_0905_2203_b200 import Context
for cfg, k in (("cfg1", None), ("cfg3", 1000)):
    types, times, a = bench.make_stream(cfg)
    full = bench.count_candidates_csr(cfg)
    eps = [full.episode(i) for i in range(k or len(full))]
    csr = bench.to_csr(eps)
    ctx = Context(0)
    ctx.load_arrays(types, times, a)
    for direction in (0, 1):
        ctx.count_tracking_csr(csr, direction)
        t0 = time.perf_counter()
        got = ctx.count_tracking_csr(csr, direction)
        t1 = time.perf_counter()
        st = ctx.last_stats
        want = ctx.count_csr(csr)
        t2 = time.perf_counter()
        print(f"{cfg} {len(eps)} eps dir {direction}: tracking {1e3*(t1-t0):.2f} ms "
              f"(device {st['total_ms']:.2f} ms), bit-sliced {1e3*(t2-t1):.2f} ms, equal={np.array_equal(got, want)}",
              flush=True)
    ctx.close()
