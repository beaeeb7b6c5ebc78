"""Shared helpers for the parity tests (test infrastructure only)."""
from __future__ import annotations

import numpy as np

from paper_0905_2203_b200 import CSR


def csr_of(episodes):
    """episodes: list of (types, [(lo, hi), ...])."""
    off = [0]
    types, lo, hi = [], [], []
    for t, cons in episodes:
        types.extend(t)
        lo.extend(c[0] for c in cons)
        hi.extend(c[1] for c in cons)
        off.append(off[-1] + len(t))
    return CSR(np.array(off, np.uint32), np.array(types, np.uint32), np.array(lo, np.int64),
               np.array(hi, np.int64))


def ep_from_json(j):
    return list(j["types"]), [tuple(c) for c in j["constraints"]]


def stream_from_json(j):
    ev = j["events"]
    types = np.array([e[0] for e in ev], dtype=np.uint32)
    times = np.array([e[1] for e in ev], dtype=np.int64)
    return types, times, int(j["alphabet"])


def fnv_u64s(values) -> str:
    h = 1469598103934665603
    for v in values:
        v = int(v)
        for b in range(8):
            h ^= (v >> (8 * b)) & 0xFF
            h = (h * 1099511628211) & ((1 << 64) - 1)
    return f"{h:016x}"


