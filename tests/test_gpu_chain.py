"""Parity of the chain map kernel (chain_impl.cuh: greedy scan of the
chain-end bitmap, prefixes shared per CTA) against the reference corpora and
the oracle port, at every forced prefix depth and segment count. The kernel
serves host-sized launches whose windows share one width (<= 16) and whose
highs are <= 32; EPI_CHAIN=1 routes sets of any size through it."""
import numpy as np
import pytest

import oracle
from helpers import csr_of
from instances import corpus

pytestmark = pytest.mark.gpu


@pytest.fixture
def chain_env(monkeypatch):
    monkeypatch.setenv("EPI_CHAIN", "1")

    def set_(depth=None, segments=None):
        for k, v in (("EPI_CHAIN_DEPTH", depth), ("EPI_FORCE_SEGMENTS", segments)):
            if v is None:
                monkeypatch.delenv(k, raising=False)
            else:
                monkeypatch.setenv(k, str(v))
    return set_


def port_counts(types, times, eps):
    c = csr_of(eps)
    return oracle.count_batch(types, times, c.offsets, c.types, c.low, c.high, threads=8)


@pytest.mark.parametrize("depth", [None, 1, 2, 3])
@pytest.mark.parametrize("segments", [None, 3, 17])
def test_chain_reference_corpora(ctx, golden_instances, chain_env, depth, segments):
    """The reference's randomised corpora (T/test_fsm.cpp, T/test_tracking.cpp,
    T/test_mapconcat.cpp, acceptance C1; windows from the (0,5],(5,10],(2,7]
    pool, i.e. width 5) through the chain kernel: == reference count_fsm."""
    chain_env(depth, segments)
    for c in golden_instances:
        gen = corpus(c["seed"], c["count"], c["max_events"], c["max_alphabet"], c["max_gap"], c["max_size"])
        for i, ((types, times, a, et, cons), want) in enumerate(zip(gen, c["instances"])):
            ctx.load_arrays(np.asarray(types, np.uint32), np.asarray(times, np.int64), a)
            got = ctx.count_csr(csr_of([(et, cons)]))
            assert int(got[0]) == want["count"], (c["name"], i, depth, segments)


def _uniform_batch(rng, a, n_eps, width, n_nodes, prefix_pool):
    """Episodes of n_nodes nodes, every window of width `width` with high in
    [width, 32], built from a small pool of prefixes so CTAs form groups."""
    pool = []
    for _ in range(prefix_pool):
        t = [int(x) for x in rng.integers(0, a, n_nodes - 1)]
        hi = [int(x) for x in rng.integers(width, 33, n_nodes - 2)] if n_nodes > 2 else []
        pool.append((t, hi))
    eps = []
    for _ in range(n_eps):
        t, hi = pool[int(rng.integers(0, len(pool)))]
        last_hi = int(rng.integers(width, 33))
        tt = t + [int(rng.integers(0, a))]
        cons = [(h - width, h) for h in hi + [last_hi]]
        eps.append((tt, cons))
    return eps


def _stream(rng, n, a, kind):
    if kind == "dense":  # many chain ends within sigma: exercises the exact check
        gaps = rng.integers(0, 3, n)
    elif kind == "bursty":  # bursts and long idle stretches (time compression)
        gaps = np.where(rng.random(n) < 0.02, rng.integers(100, 5000, n), rng.integers(0, 6, n))
    else:
        gaps = rng.integers(0, 12, n)
    return rng.integers(0, a, n).astype(np.uint32), np.cumsum(gaps).astype(np.int64)


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("kind", ["dense", "bursty", "sparse"])
def test_chain_uniform_batches_vs_port(ctx, chain_env, seed, kind):
    rng = np.random.default_rng(7000 + seed)
    a = int(rng.integers(2, 12))
    types, times = _stream(rng, int(rng.integers(500, 20000)), a, kind)
    ctx.load_arrays(types, times, a)
    for n_nodes in (2, 3, 4, 5, 8):
        width = int(rng.integers(1, 17))
        eps = _uniform_batch(rng, a, int(rng.integers(20, 700)), width, n_nodes, int(rng.integers(1, 12)))
        want = port_counts(types, times, eps)
        for depth in (None, 1, 2, n_nodes):
            for segments in (None, 5):
                chain_env(depth, segments)
                got = ctx.count_csr(csr_of(eps))
                np.testing.assert_array_equal(got, want, err_msg=f"{kind} N={n_nodes} W={width} d={depth} P={segments}")


def test_chain_default_threshold_and_knob(ctx, monkeypatch):
    """Sets of >= 1024 episodes take the chain kernel by default; EPI_CHAIN=0
    keeps the automaton kernel: both equal the port."""
    rng = np.random.default_rng(5)
    types, times = _stream(rng, 60000, 16, "sparse")
    ctx.load_arrays(types, times, 16)
    eps = _uniform_batch(rng, 16, 3000, 5, 3, 40)
    want = port_counts(types, times, eps)
    np.testing.assert_array_equal(ctx.count_csr(csr_of(eps)), want)
    monkeypatch.setenv("EPI_CHAIN", "0")
    np.testing.assert_array_equal(ctx.count_csr(csr_of(eps)), want)


def test_chain_two_pass_mode(ctx, chain_env):
    """MODE_MINE batches: pass 2 of the hull relaxation counts host-sized
    survivor sets through the chain kernel; counts of survivors stay exact."""
    from paper_0905_2203_b200 import COUNT_PRUNED, MODE_MINE
    rng = np.random.default_rng(11)
    types, times = _stream(rng, 30000, 6, "sparse")
    ctx.load_arrays(types, times, 6)
    eps = _uniform_batch(rng, 6, 2000, 5, 3, 30)
    want = port_counts(types, times, eps)
    got = ctx.count_csr(csr_of(eps), threshold=int(np.median(want)), mode=MODE_MINE)
    keep = got != np.uint64(COUNT_PRUNED)
    np.testing.assert_array_equal(got[keep], want[keep])
    assert np.all(want[~keep] < int(np.median(want)))


@pytest.mark.parametrize("dedup", [True, False])
def test_chain_duplicate_episodes(ctx, chain_env, monkeypatch, dedup):
    """Identical episodes are counted once (distinct episodes gathered after
    the sort, counts scattered back to every caller slot); EPI_NO_DEDUP
    counts every copy."""
    if not dedup:
        monkeypatch.setenv("EPI_NO_DEDUP", "1")
    rng = np.random.default_rng(21)
    types, times = _stream(rng, 40000, 8, "sparse")
    ctx.load_arrays(types, times, 8)
    base = _uniform_batch(rng, 8, 300, 5, 3, 6)
    eps = [base[int(i)] for i in rng.integers(0, len(base), 5000)]
    want = port_counts(types, times, base)
    got = ctx.count_csr(csr_of(eps))
    index = {(tuple(t), tuple(c)): i for i, (t, c) in enumerate(base)}
    np.testing.assert_array_equal(got, [want[index[(tuple(t), tuple(c))]] for t, c in eps])


@pytest.mark.parametrize("kind", ["sparse", "dense", "bursty"])
def test_mine_mode_popcount_pass1(ctx, kind):
    """epi_count MODE_MINE on a uniform batch: pass 1 is the device
    chain-end popcount bound (sound: every completion is a distinct chain
    end), pass 2 the exact count of the survivors; the frequent set equals
    the exact one and no frequent candidate is pruned. EPI_PASS1_HULL keeps
    the host hull relaxation."""
    from paper_0905_2203_b200 import COUNT_PRUNED, MODE_MINE
    rng = np.random.default_rng(31)
    types, times = _stream(rng, 30000, 6, kind)
    ctx.load_arrays(types, times, 6)
    eps = _uniform_batch(rng, 6, 3000, 5, 3, 30)
    want = port_counts(types, times, eps)
    thr = max(2, int(np.percentile(want, 80)))
    got, freq = ctx.count_csr(csr_of(eps), threshold=thr, mode=MODE_MINE, with_frequent=True)
    keep = got != np.uint64(COUNT_PRUNED)
    np.testing.assert_array_equal(got[keep], want[keep])
    assert np.all(want[~keep] < thr)
    np.testing.assert_array_equal(freq.astype(bool), want >= thr)
    st = ctx.last_stats
    assert st["pass1_groups"] == len(eps) and st["pruned"] == int((~keep).sum())
    assert st["chain_launches"] >= 1


@pytest.mark.parametrize("alphabet", [120, 300])
def test_chain_large_alphabet_two_stage_ring(ctx, chain_env, alphabet):
    """Alphabets whose bitmap blocks no longer fit three (or four) staging
    buffers: the chain kernel runs with the 2-deep ring."""
    rng = np.random.default_rng(alphabet)
    types, times = _stream(rng, 200_000, alphabet, "sparse")
    ctx.load_arrays(types, times, alphabet)
    eps = _uniform_batch(rng, alphabet, 5000, 5, 3, 200)
    want = port_counts(types, times, eps)
    for depth in (None, 1, 3):
        chain_env(depth)
        np.testing.assert_array_equal(ctx.count_csr(csr_of(eps)), want)


@pytest.mark.parametrize("n_nodes", [6, 7, 8])
def test_chain_long_episodes_large_sets(ctx, n_nodes, monkeypatch):
    """Long episodes in sets large enough for the default chain path, the
    dedup and the 4-deep ring (>= 65,536 episodes), against the port on a
    subset and against the automaton kernel on all of them."""
    rng = np.random.default_rng(n_nodes)
    types, times = _stream(rng, 100_000, 6, "dense")
    ctx.load_arrays(types, times, 6)
    eps = _uniform_batch(rng, 6, 70_000, 3, n_nodes, 400)
    got = ctx.count_csr(csr_of(eps))
    assert ctx.last_stats["chain_launches"] >= 1
    np.testing.assert_array_equal(got[:300], port_counts(types, times, eps[:300]))
    monkeypatch.setenv("EPI_CHAIN", "0")
    np.testing.assert_array_equal(got, ctx.count_csr(csr_of(eps)))
