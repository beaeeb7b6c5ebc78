"""Parallel local tracking on the device (epi_find_occurrences /
epi_count_tracking) against the reference: the occurrence intervals must be
the reference's find_occurrences output exactly (order included), both
directions; counts must equal count_fsm. At scale, the two device counters
(tracking and the bit-sliced automaton) cross-check each other."""
import numpy as np
import pytest

import oracle
from helpers import csr_of, ep_from_json
from instances import corpus
from paper_0905_2203_b200 import GenConfig, generate_arrays

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="reference build (oracle/_ref) absent")


def load(ctx, types, times, a):
    ctx.load_arrays(np.asarray(types, np.uint32), np.asarray(times, np.int64), a)


def device_intervals(ctx, eps, direction):
    off, s, e = ctx.find_occurrences_csr(csr_of(eps), direction)
    return [list(zip(s[off[i]:off[i + 1]].tolist(), e[off[i]:off[i + 1]].tolist())) for i in range(len(eps))]


@pytest.mark.parametrize("direction", [0, 1])
def test_tracking_known_answers(ctx, direction):
    """T/test_tracking.cpp:45-67, 128-136, 161-176."""
    load(ctx, [0, 1, 2], [1, 8, 20], 3)
    assert device_intervals(ctx, [([0, 1, 2], [(5, 10), (10, 15)])], direction) == [[(1, 20)]]
    load(ctx, [0, 1, 0], [2, 3, 7], 2)
    assert device_intervals(ctx, [([0], [])], direction) == [[(2, 2), (7, 7)]]
    load(ctx, [0, 0, 1], [0, 2, 6], 2)
    assert list(ctx.count_tracking_csr(csr_of([([0, 1], [(0, 10)])]), direction)) == [1]
    load(ctx, [0] + [1] * 9, list(range(10)), 2)
    # forward: one interval per reached B (the reference's 9); backward: one
    # per reached A, keeping the earliest end
    want = [(0, t) for t in range(1, 10)] if direction == 0 else [(0, 1)]
    assert device_intervals(ctx, [([0, 1], [(0, 10)])], direction)[0] == want
    assert list(ctx.count_tracking_csr(csr_of([([0, 1], [(0, 10)])]), direction)) == [1]


@needs_ref
@pytest.mark.parametrize("direction", [0, 1])
def test_tracking_corpus_vs_reference(ctx, golden_instances, direction):
    """T/test_tracking.cpp:225-242 corpus (seed 62) and acceptance C1: the
    interval lists equal the reference's, the counts equal count_fsm."""
    for c in golden_instances:
        if c["name"] not in ("tracking_vs_oracle", "acceptance_c1"):
            continue
        gen = corpus(c["seed"], c["count"], c["max_events"], c["max_alphabet"], c["max_gap"], c["max_size"])
        for i, ((types, times, a, et, cons), want) in enumerate(zip(gen, c["instances"])):
            load(ctx, types, times, a)
            got = device_intervals(ctx, [(et, cons)], direction)[0]
            ref = oracle.ref_find_occurrences(types, times, a, et, [x[0] for x in cons], [x[1] for x in cons],
                                              direction)
            assert got == ref, (c["name"], i, direction)
            assert int(ctx.count_tracking_csr(csr_of([(et, cons)]), direction)[0]) == want["count"]


@needs_ref
@pytest.mark.parametrize("seed", range(3))
def test_tracking_random_vs_reference(ctx, seed):
    rng = np.random.default_rng(7000 + seed)
    for it in range(15):
        n = int(rng.integers(0, 4000))
        a = int(rng.integers(1, 7))
        times = np.cumsum(rng.integers(0, [2, 6, 30][it % 3] + 1, n)).astype(np.int64)
        types = rng.integers(0, a, n).astype(np.uint32)
        eps = []
        for _ in range(12):
            N = int(rng.integers(1, 6))
            cons = []
            for _k in range(N - 1):
                h = int(rng.integers(1, 40))
                cons.append((int(rng.integers(0, h)), h))
            eps.append(([int(x) for x in rng.integers(0, a, N)], cons))
        load(ctx, types, times, a)
        for direction in (0, 1):
            got = device_intervals(ctx, eps, direction)
            for j, (et, cons) in enumerate(eps):
                ref = oracle.ref_find_occurrences(types, times, a, et, [x[0] for x in cons],
                                                  [x[1] for x in cons], direction)
                assert got[j] == ref, (seed, it, j, direction)
        csr = csr_of(eps)
        want = oracle.count_batch(types, times, csr.offsets, csr.types, csr.low, csr.high)
        for direction in (0, 1):
            np.testing.assert_array_equal(ctx.count_tracking_csr(csr, direction), want)


def test_tracking_cross_checks_bitsliced_on_cfg3(ctx, golden_configs):
    """cfg3 (10M events): the first 256 candidates' tracking counts equal the
    reference's; 1,000 more cross-check the two device counters."""
    g = golden_configs["cfg3"]
    types, times = generate_arrays(GenConfig(64, 7813, 20, [], 3))
    ctx.load_arrays(types, times, 64)
    eps = [ep_from_json(e) for e in g["episodes"]]
    assert [int(x) for x in ctx.count_tracking_csr(csr_of(eps), 1)] == g["counts"]
    rng = np.random.default_rng(12)
    more = [([int(x) for x in rng.integers(0, 64, 3)], [(0, 5), (5, 10)]) for _ in range(1000)]
    csr = csr_of(more)
    np.testing.assert_array_equal(ctx.count_tracking_csr(csr, 0), ctx.count_csr(csr))


@needs_ref
@pytest.mark.parametrize("direction", [0, 1])
def test_tracking_stats_vs_reference(ctx, golden_instances, direction):
    """TrackingStats analogue: items_tracked == the number of occurrence
    intervals the reference's find_occurrences returns (E/tracking.hpp:353);
    no sort fallback on these corpora (T/test_tracking.cpp:178-192)."""
    for c in golden_instances[:2]:
        gen = corpus(c["seed"], min(c["count"], 60), c["max_events"], c["max_alphabet"], c["max_gap"],
                     c["max_size"])
        for (types, times, a, et, cons) in gen:
            load(ctx, types, times, a)
            got = ctx.count_tracking_csr(csr_of([(et, cons)]), direction)
            st = ctx.last_stats
            ref = oracle.ref_find_occurrences(types, times, a, et, [x[0] for x in cons], [x[1] for x in cons],
                                              direction)
            assert st["items_tracked"] == len(ref)
            assert st["sort_fallbacks"] == 0
            assert int(got[0]) == oracle.count_fsm(types, times, et, [x[0] for x in cons], [x[1] for x in cons])


def test_count_mapconcat_segments(ctx, golden_instances):
    """count_mapconcat with the caller's segment count (epi_count_mapconcat):
    the count never depends on it (T/test_mapconcat.cpp:137-145) and the
    segments used are reported (clamped to what the stream allows)."""
    from paper_0905_2203_b200 import EventStream, Episode, MapConcatStats, count_mapconcat
    c = golden_instances[0]
    gen = corpus(c["seed"], 40, c["max_events"], c["max_alphabet"], c["max_gap"], c["max_size"])
    for (types, times, a, et, cons), want in zip(gen, c["instances"]):
        load(ctx, types, times, a)
        for P in (1, 2, 5, 64):
            got = ctx.count_mapconcat_csr(csr_of([(et, cons)]), P)
            assert int(got[0]) == want["count"]
            assert 1 <= ctx.last_stats["segments"] <= P
        st = MapConcatStats()
        s = EventStream(np.asarray(types, np.uint32), np.asarray(times, np.int64), a)
        assert count_mapconcat(s, Episode(et, cons), 3, stats=st) == want["count"]
        assert st.machine_hits + st.patches == st.machines_precomputed >= 1
