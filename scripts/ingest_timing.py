"""Stream ingest timings: binary event file
(epi_load_stream_file: mapped, pinned double-buffered H2D) vs host arrays
(epi_load_stream) vs the text format (epi_parse_events + epi_load_stream).
The file is written first, so it is read from the page cache."""
import os, sys, time, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_0905_2203_b200 import Context, write_events_binary, load_stream, serialize_stream, EventStream

def best(f, k=3):
    ts = []
    for _ in range(k):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    return min(ts)

ctx = Context(0)
rng = np.random.default_rng(0)
for n in (10_000_000, 100_000_000):
    types = rng.integers(0, 64, n).astype(np.uint32)
    times = np.cumsum(rng.integers(0, 2, n)).astype(np.int64)
    d = tempfile.mkdtemp()
    p = os.path.join(d, "s.evt")
    t_w = best(lambda: write_events_binary(p, types, times, 64), 1)
    t_f = best(lambda: ctx.load_file(p))
    t_a = best(lambda: ctx.load_arrays(types, times, 64))
    gb = n * 12 / 1e9
    print(f"n={n:>11,}  write {t_w*1e3:8.1f} ms   load_file {t_f*1e3:8.1f} ms ({gb/t_f:5.1f} GB/s)   "
          f"load_arrays {t_a*1e3:8.1f} ms ({gb/t_a:5.1f} GB/s)")
    os.remove(p)
n = 10_000_000
types = rng.integers(0, 64, n).astype(np.uint32)
times = np.cumsum(rng.integers(0, 2, n)).astype(np.int64)
text = "".join(f"n{t},{tm}\n" for t, tm in zip(types[:2_000_000].tolist(), times[:2_000_000].tolist()))
t_p = best(lambda: load_stream(text), 2)
print(f"text 2,000,000 events ({len(text)/1e6:.0f} MB): parse {t_p*1e3:.1f} ms ({2e6/t_p/1e6:.0f} M events/s)")
