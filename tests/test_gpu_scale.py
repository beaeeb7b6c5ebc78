"""Parity at the BASELINE.json scales (configs 3-5) against the REFERENCE:
tests/golden/scale.json holds counts computed by the unmodified reference
(oracle/_ref, count_fsm on all host cores; oracle/make_scale_golden.py) on
the full-size streams:
  * cfg3: every one of the 10,000 candidates;
  * cfg4 (MEA-shaped, ~100M events): the first 1,000 seeded 5-node
    candidates + the two embedded chains;
  * cfg5 cells (1M .. 1B events): the first 1,000 candidates of the seeded
    sequence every cell draws from (so the subset of every |C| cell, up to
    the 10M x 1M headline cell).
Plus size-independent properties of the counting semantics on every
candidate of a cell:
  * idempotent ties: duplicating every event leaves every count unchanged
    (same-type ties collapse);
  * time-shift invariance: adding a constant to every timestamp;
  * gap invariance: stretching every gap longer than the largest window;
  * prefix monotonicity: a prefix never counts more than the whole stream.
"""
import json
import os

import numpy as np
import pytest

import oracle
from helpers import csr_of
from paper_0905_2203_b200 import (BurstConfig, Embedding, Episode, GenConfig, generate_arrays,
                                  generate_bursty_arrays, random_episodes_csr)

pytestmark = pytest.mark.gpu

BINS = [(0, 5), (5, 10), (10, 15)]
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "scale.json")


@pytest.fixture(scope="module")
def scale():
    with open(GOLDEN) as f:
        return json.load(f)


def stream_of(cell, ctx=None):
    s = cell["stream"]
    if s["kind"] == "generate" and ctx is not None:
        # the device generator (bit-exact generate(); tests/test_gpu_datagen.py)
        ctx.generate(GenConfig(s["neurons"], s["duration_s"], s["rate_hz"], [], s["seed"]))
        types, times = ctx.download()
    elif s["kind"] == "generate":
        types, times = generate_arrays(GenConfig(s["neurons"], s["duration_s"], s["rate_hz"], [], s["seed"]))
    else:
        emb = [Embedding(Episode(t, [tuple(c) for c in cs]), s["embedded_rate_hz"]) for t, cs in cell["extra"]]
        bc = BurstConfig(electrodes=s["electrodes"], duration_s=s["duration_s"], seed=s["seed"], embedded=emb)
        if ctx is not None:
            ctx.generate_bursty(bc)
            types, times = ctx.download()
        else:
            types, times = generate_bursty_arrays(bc)
    assert len(types) == cell["n"]
    assert oracle.fnv_stream(types, times, cell["alphabet"]) == cell["stream_fnv"]
    return types, times


def cands_of(cell, count=None):
    c = cell["cands"]
    csr = random_episodes_csr(c["seed"], count or c["count"], c["nodes"], c["alphabet"], BINS)
    if cell["extra"] and count is None:
        extra = csr_of([(t, [tuple(x) for x in cs]) for t, cs in cell["extra"]])
        off = np.concatenate([csr.offsets, csr.offsets[-1] + extra.offsets[1:]])
        from paper_0905_2203_b200 import CSR
        csr = CSR(off, np.concatenate([csr.types, extra.types]), np.concatenate([csr.low, extra.low]),
                  np.concatenate([csr.high, extra.high]))
    return csr


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


def test_scale_candidates_match_reference_draws(scale):
    """The product's seeded candidate generator == the fixture's draws
    (pure-Python mt19937_64 in the reference's order)."""
    for name in ("cfg3", "cfg4", "cfg5_1000000"):
        c = scale[name]["cands"]
        eps = oracle.mt_episodes(c["seed"], 50, c["nodes"], c["alphabet"], BINS)
        got = cands_of(scale[name], 50)
        np.testing.assert_array_equal(got.types, np.concatenate([t for t, _ in eps]))
        np.testing.assert_array_equal(got.high, np.array([x[1] for _, cs in eps for x in cs]))


@pytest.mark.parametrize("kernel", ["chain", "automaton"])
def test_cfg3_all_candidates(ctx, scale, kernel, monkeypatch):
    """cfg3: all 10,000 candidates == the reference's count_fsm."""
    if kernel == "automaton":
        monkeypatch.setenv("EPI_CHAIN", "0")
    cell = scale["cfg3"]
    types, times = stream_of(cell, ctx)
    got = ctx.count_csr(cands_of(cell))
    want = np.array(cell["counts"], np.uint64)
    bad = np.nonzero(got != want)[0]
    assert len(bad) == 0, f"{len(bad)} mismatches, first {bad[:5].tolist()}"
    assert int(got.sum()) == cell["sum"]


def test_cfg4_mea_bursty_100m(ctx, scale):
    """cfg4: the first 1,000 seeded 5-node candidates + the embedded chains
    over ~100M bursty events == the reference; properties on all of them."""
    cell = scale["cfg4"]
    types, times = stream_of(cell, ctx)
    csr = cands_of(cell)
    got = ctx.count_csr(csr)
    np.testing.assert_array_equal(got, np.array(cell["counts"], np.uint64))
    assert int(got[-1]) > 0 and int(got[-2]) > 0
    properties(ctx, types, times, cell["alphabet"], csr, got)


@pytest.mark.parametrize("n_events,n_cands", [(1_000_000, 1000), (10_000_000, 10_000), (10_000_000, 1_000_000),
                                              (100_000_000, 10_000), (1_000_000_000, 1000)])
def test_cfg5_sweep_cells(ctx, scale, n_events, n_cands):
    """cfg5 cells: the cell's first 1,000 candidates == the reference; the
    properties on every candidate of the smaller cells."""
    name = f"cfg5_{n_events}"
    if name not in scale:
        pytest.skip(f"{name} not in the scale fixture")
    cell = scale[name]
    types, times = stream_of(cell, ctx)  # generated on the device, already loaded
    csr = cands_of(cell, n_cands)
    got = ctx.count_csr(csr)
    np.testing.assert_array_equal(got[:1000], np.array(cell["counts"], np.uint64))
    if n_events * n_cands <= 1e11:
        properties(ctx, types, times, cell["alphabet"], csr, got)
