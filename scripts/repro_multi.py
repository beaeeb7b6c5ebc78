import sys
import numpy as np
sys.path.insert(0, ".")
from paper_0905_2203_b200 import Context, EventStream, MiningConfig, mine, write_mining_csv, MODE_MINE
rng = np.random.default_rng(84)
n = 3000
types = rng.integers(0, 6, n).astype(np.uint32)
times = np.cumsum(rng.integers(0, 3, n)).astype(np.int64)
cfg = MiningConfig(threshold=5, constraint_alphabet=[(0, 5), (5, 10)], max_level=4, mode=MODE_MINE)
one = Context(0)
want = mine(EventStream(types, times, 6), cfg, ctx=one)
print("levels", [lv.candidates for lv in want.levels], flush=True)
m = Context(devices=[0, 0])
got = mine(EventStream(types, times, 6), cfg, ctx=m)
print("multi levels", [lv.candidates for lv in got.levels], flush=True)
print("equal", write_mining_csv(got) == write_mining_csv(want), flush=True)
