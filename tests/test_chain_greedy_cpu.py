"""DESIGN.md §1's chain-end greedy, restated on 32 ms bitmap tiles in plain
Python and checked against the oracle port (run_fsm, E/fsm.hpp:45-106).

The chain kernel (paper_0905_2203_b200/csrc/chain_impl.cuh) counts by a
greedy scan of U_{N-1}, the bitmap of chain ends: after a completion at pe,
bits in (pe, pe + L] are never completions, the first bit after pe + sigma
always is, and a bit in (pe + L, pe + sigma] needs an exact check. This test
pins that argument with the simplest exact check - rebuild the chain bitmaps
from starts after pe, whose first chain end is the next completion - on
dense and sparse random streams, so the basis of the device kernel is
checked independently of the device."""
import numpy as np
import pytest

import oracle


def _window_any(c, h1, lo1, hi):
    # bit i: a bit of (c : h1) at age a in [lo1, hi] from time 32g + i
    x = (c << 32) | h1
    r = 0
    for i in range(32):
        for a in range(lo1, hi + 1):
            j = 32 + i - a
            if j >= 0 and (x >> j) & 1:
                r |= 1 << i
                break
    return r


def greedy_count(types, times, ep, cons):
    n_tiles = (int(times.max()) + 1 + 31) // 32 + 2 if len(times) else 2
    occ = {}
    for ty, t in zip(types.tolist(), times.tolist()):
        row = occ.setdefault(ty, [0] * n_tiles)
        row[t >> 5] |= 1 << (t & 31)
    zero = [0] * n_tiles
    rows = [occ.get(ty, zero) for ty in ep]
    lo1 = [c[0] + 1 for c in cons]
    hi = [c[1] for c in cons]
    sigma, big_l, n = sum(hi), sum(lo1), len(ep)
    st = {"pe": -1, "floor": -1, "ready": -1, "cnt": 0}

    def chain_word(g, hist, mask):
        cw = rows[0][g] & mask
        for k in range(1, n):
            nx = rows[k][g] & _window_any(cw, hist[k - 1], lo1[k - 1], hi[k - 1])
            hist[k - 1] = cw
            cw = nx
        return cw

    def validate():
        start, lim = st["pe"] + 1, st["pe"] + sigma
        hist = [0] * (n - 1)
        mask = (0xFFFFFFFF << (start & 31)) & 0xFFFFFFFF
        for g in range(start >> 5, min((lim >> 5) + 1, n_tiles)):
            cw = chain_word(g, hist, mask)
            mask = 0xFFFFFFFF
            if cw:
                t = 32 * g + (cw & -cw).bit_length() - 1
                st.update(cnt=st["cnt"] + 1, pe=t, floor=t + big_l, ready=t + sigma)
                return
        st["floor"] = st["ready"] = st["pe"] + sigma

    def above(f, base):
        d = f - base
        return 0xFFFFFFFF if d < 0 else (0 if d >= 31 else (0xFFFFFFFF << (d + 1)) & 0xFFFFFFFF)

    hist = [0] * (n - 1)
    for g in range(n_tiles):
        w = chain_word(g, hist, 0xFFFFFFFF) & above(st["floor"], 32 * g)
        while w:
            t = 32 * g + (w & -w).bit_length() - 1
            if t > st["ready"]:
                st.update(cnt=st["cnt"] + 1, pe=t, floor=t + big_l, ready=t + sigma)
            else:
                validate()
            w &= above(st["floor"], 32 * g)
    return st["cnt"]


@pytest.mark.parametrize("kind", ["dense", "sparse"])
def test_chain_end_greedy_equals_run_fsm(kind):
    rng = np.random.default_rng(4242 if kind == "dense" else 4243)
    for _ in range(25):
        a = int(rng.integers(2, 6))
        n_ev = int(rng.integers(50, 250))
        gaps = rng.integers(0, 3, n_ev) if kind == "dense" else rng.integers(0, 12, n_ev)
        types = rng.integers(0, a, n_ev).astype(np.uint32)
        times = np.cumsum(gaps).astype(np.int64)
        nodes = int(rng.choice([2, 3, 5]))
        width = int(rng.integers(1, 17))
        ep = [int(x) for x in rng.integers(0, a, nodes)]
        cons = []
        for _k in range(nodes - 1):
            h = int(rng.integers(width, 33))
            cons.append((h - width, h))
        want = oracle.count_fsm(types, times, ep, [c[0] for c in cons], [c[1] for c in cons])
        assert greedy_count(types, times, ep, cons) == want, (ep, cons)
