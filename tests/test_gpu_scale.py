"""Parity at the BASELINE.json scales (configs 3-5): seeded candidate subsets
against the oracle port on the full streams, plus size-independent
properties of the counting semantics checked on every candidate:
  * idempotent ties: duplicating every event leaves every count unchanged
    (same-type ties collapse);
  * time-shift invariance: adding a constant to every timestamp;
  * gap invariance: stretching every gap longer than the largest window;
  * prefix monotonicity: a prefix never counts more than the whole stream.
"""
import numpy as np
import pytest

import oracle
from helpers import csr_of
from paper_0905_2203_b200 import BurstConfig, Embedding, Episode, GenConfig, generate_arrays, generate_bursty_arrays

pytestmark = pytest.mark.gpu

BINS = [(0, 5), (5, 10), (10, 15)]


def random_candidates(rng, n, alphabet, nodes):
    return [([int(x) for x in rng.integers(0, alphabet, nodes)],
             [BINS[int(b)] for b in rng.integers(0, 3, nodes - 1)]) for _ in range(n)]


def check_subset(types, times, eps, got, k, seed):
    rng = np.random.default_rng(seed)
    pick = np.sort(rng.choice(len(eps), size=min(k, len(eps)), replace=False))
    sub = csr_of([eps[i] for i in pick])
    want = oracle.count_batch(types, times, sub.offsets, sub.types, sub.low, sub.high, threads=16)
    np.testing.assert_array_equal(got[pick], want)


def properties(ctx, types, times, alphabet, csr, base):
    # duplicated events (ties)
    ctx.load_arrays(np.repeat(types, 2), np.repeat(times, 2), alphabet)
    np.testing.assert_array_equal(ctx.count_csr(csr), base)
    # time shift
    ctx.load_arrays(types, times + 123_456_789, alphabet)
    np.testing.assert_array_equal(ctx.count_csr(csr), base)
    # stretch gaps above the largest window (high <= 15 here)
    gaps = np.diff(times, prepend=times[:1])
    stretched = np.cumsum(np.where(gaps > 20, gaps * 3, gaps)).astype(np.int64)
    ctx.load_arrays(types, stretched, alphabet)
    np.testing.assert_array_equal(ctx.count_csr(csr), base)
    # prefix monotonicity
    half = len(types) // 2
    ctx.load_arrays(types[:half], times[:half], alphabet)
    assert np.all(ctx.count_csr(csr) <= base)


def test_cfg3_full_stream_properties(ctx):
    """cfg3: 10,004,428 events, 64 types; 2,000 seeded 3-node candidates."""
    types, times = generate_arrays(GenConfig(64, 7813, 20, [], 3))
    rng = np.random.default_rng(33)
    eps = random_candidates(rng, 2000, 64, 3)
    csr = csr_of(eps)
    ctx.load_arrays(types, times, 64)
    base = ctx.count_csr(csr)
    check_subset(types, times, eps, base, 48, 1)
    properties(ctx, types, times, 64, csr, base)


def test_cfg4_mea_bursty_100m(ctx):
    """cfg4: MEA-shaped, 60 electrodes, ~100M events with network bursts;
    5-node candidates (random + the embedded chains)."""
    chains = [Episode([0, 7, 13, 21, 33], [(5, 10), (0, 5), (10, 15), (5, 10)]),
              Episode([40, 41, 42, 43, 44], [(0, 5)] * 4)]
    cfg = BurstConfig(electrodes=60, duration_s=175_000, seed=4,
                      embedded=[Embedding(c, 0.5) for c in chains])
    types, times = generate_bursty_arrays(cfg)
    assert 90e6 < len(types) < 110e6
    rng = np.random.default_rng(44)
    eps = random_candidates(rng, 2046, 60, 5) + [(c.types, c.constraints) for c in chains]
    ctx.load_arrays(types, times, 60)
    got = ctx.count_csr(csr_of(eps))
    check_subset(types, times, eps, got, 40, 2)
    tail = csr_of(eps[-2:])
    want = oracle.count_batch(types, times, tail.offsets, tail.types, tail.low, tail.high, threads=2)
    np.testing.assert_array_equal(got[-2:], want)
    assert int(got[-1]) > 0 and int(got[-2]) > 0


@pytest.mark.parametrize("n_events,n_cands", [(1_000_000, 1000), (10_000_000, 10000), (100_000_000, 1000)])
def test_cfg5_sweep_cells(ctx, n_events, n_cands):
    """cfg5 cells: 64 types at 20 Hz, random 3-node x 3-bin candidates."""
    duration = n_events / (64 * 20)
    types, times = generate_arrays(GenConfig(64, duration, 20, [], 5 + n_events))
    rng = np.random.default_rng(n_events + n_cands)
    eps = random_candidates(rng, n_cands, 64, 3)
    ctx.load_arrays(types, times, 64)
    got = ctx.count_csr(csr_of(eps))
    check_subset(types, times, eps, got, 24 if n_events >= 100_000_000 else 64, 3)
