"""Parity of the B200 counting path (through the C-ABI) against the reference:
golden known-answer tests, the reference's randomised corpora, the bench
configs, and the oracle port on larger random instances. Bit-exact (integer
counts), no tolerance."""
import os

import numpy as np
import pytest

import oracle
from helpers import csr_of, ep_from_json, stream_from_json, fnv_u64s
from instances import corpus
from paper_0905_2203_b200 import (COUNT_PRUNED, MODE_EXACT, MODE_MINE, DataError, Embedding, Episode,
                                  GenConfig, InvalidArgument, Unsupported, generate_arrays)

pytestmark = pytest.mark.gpu

BINS = [(0, 5), (5, 10), (10, 15)]


def count_one(ctx, types, times, alphabet, eps, **kw):
    ctx.load_arrays(np.asarray(types, np.uint32), np.asarray(times, np.int64), alphabet)
    return ctx.count_csr(csr_of(eps), **kw)


@pytest.fixture
def segments_env():
    old = os.environ.get("EPI_FORCE_SEGMENTS")

    def set_(v):
        if v is None:
            os.environ.pop("EPI_FORCE_SEGMENTS", None)
        else:
            os.environ["EPI_FORCE_SEGMENTS"] = str(v)
    yield set_
    set_(old)


def test_known_answer_tests(ctx, golden_kats):
    for k in golden_kats["count"]:
        types, times, a = stream_from_json(k)
        got = count_one(ctx, types, times, a, [ep_from_json(k["episode"])])
        assert int(got[0]) == k["expected"] == k["count_fsm"], k["name"]


def test_known_answer_tests_many_segments(ctx, golden_kats, segments_env):
    for p in (2, 3, 7, 64):
        segments_env(p)
        for k in golden_kats["count"]:
            types, times, a = stream_from_json(k)
            got = count_one(ctx, types, times, a, [ep_from_json(k["episode"])])
            assert int(got[0]) == k["expected"], (k["name"], p)


@pytest.fixture(params=["warp", "seq"])
def walk_mode(request, monkeypatch):
    """Concat walk: warp-parallel (default for small sets) or the sequential
    one-thread-per-episode walk (EPI_WALK_SEQ)."""
    if request.param == "seq":
        monkeypatch.setenv("EPI_WALK_SEQ", "1")
    return request.param


@pytest.mark.parametrize("force", [None, 2, 5, 13, 64])
def test_reference_corpora(ctx, golden_instances, segments_env, force, walk_mode):
    """T/test_fsm.cpp, T/test_tracking.cpp, T/test_mapconcat.cpp,
    T/acceptance.cpp C1 corpora: device count == reference count_fsm ==
    oracle_count, at several forced segment counts (MapConcatenate
    P-independence, cf. T/test_mapconcat.cpp:137-145)."""
    segments_env(force)
    for c in golden_instances:
        gen = corpus(c["seed"], c["count"], c["max_events"], c["max_alphabet"], c["max_gap"],
                     c["max_size"])
        for i, ((types, times, a, et, cons), want) in enumerate(zip(gen, c["instances"])):
            got = count_one(ctx, types, times, a, [(et, cons)])
            assert int(got[0]) == want["count"], (c["name"], i, force)


def _random_case(rng, n_max, alphabet_max, gap_max, n_nodes_max, high_max):
    n = int(rng.integers(0, n_max + 1))
    a = int(rng.integers(1, alphabet_max + 1))
    times = np.cumsum(rng.integers(0, gap_max + 1, size=n)).astype(np.int64)
    types = rng.integers(0, a, size=n).astype(np.uint32)
    eps = []
    for _ in range(int(rng.integers(1, 40))):
        N = int(rng.integers(1, n_nodes_max + 1))
        et = [int(x) for x in rng.integers(0, a, size=N)]
        cons = []
        for _k in range(N - 1):
            hi = int(rng.integers(1, high_max + 1))
            lo = int(rng.integers(0, hi))
            cons.append((lo, hi))
        eps.append((et, cons))
    return types, times, a, eps


@pytest.mark.parametrize("seed", range(6))
def test_random_vs_port(ctx, seed, segments_env, walk_mode):
    """Wider random instances than the reference's (windows up to 63, up to
    10 nodes, thousands of events, idle gaps that trigger time compression)
    against the oracle port (count_fsm restated)."""
    rng = np.random.default_rng(1000 + seed)
    for it in range(60):
        segments_env([None, 3, 11][it % 3])
        gap_max = [3, 12, 90][it % 3]
        types, times, a, eps = _random_case(rng, 3000, 8, gap_max, 10, 63)
        got = count_one(ctx, types, times, a, eps)
        csr = csr_of(eps)
        want = oracle.count_batch(types, times, csr.offsets, csr.types, csr.low, csr.high, threads=4)
        np.testing.assert_array_equal(got, want, err_msg=f"seed {seed} it {it}")


def test_edge_cases(ctx):
    # empty stream
    assert list(count_one(ctx, [], [], 3, [([0, 1], [(0, 5)]), ([2], [])])) == [0, 0]
    # every event at one timestamp: nothing chains; singletons collapse
    got = count_one(ctx, [0, 1, 0, 1], [7, 7, 7, 7], 2, [([0, 1], [(0, 5)]), ([0], []), ([1], [])])
    assert list(got) == [0, 1, 1]
    # types outside the alphabet never fire (count_fsm returns 0)
    got = count_one(ctx, [0, 1], [0, 7], 2, [([0, 5], [(5, 10)]), ([9], [])])
    assert list(got) == [0, 0]
    # high = 63 exactly at the edge, across a tile boundary
    got = count_one(ctx, [0, 1, 0, 1], [0, 63, 70, 134], 2, [([0, 1], [(0, 63)]), ([0, 1], [(62, 63)])])
    assert list(got) == [1, 1]
    # 16-node episode with repeated types
    ev_t = [i % 3 for i in range(400)]
    ev_tm = list(range(0, 1200, 3))
    ep = ([0, 1, 2] * 5 + [0], [(0, 5)] * 15)
    got = count_one(ctx, ev_t, ev_tm, 3, [ep])
    assert int(got[0]) == oracle.count_fsm(ev_t, ev_tm, ep[0], [c[0] for c in ep[1]], [c[1] for c in ep[1]])
    # long idle gaps (compression) and times far from zero
    t0 = 10**12
    got = count_one(ctx, [0, 1, 0, 1], [t0, t0 + 7, t0 + 10**9, t0 + 10**9 + 6], 2, [([0, 1], [(5, 10)])])
    assert int(got[0]) == 2


def test_binary_event_file_load(ctx, tmp_path):
    """epi_load_stream_file (mapped binary file) == epi_load_stream (arrays):
    same counts, same validation messages."""
    from paper_0905_2203_b200 import generate_arrays, GenConfig, write_events_binary
    types, times = generate_arrays(GenConfig(neurons=12, duration_s=20, base_rate_hz=30, seed=3))
    rng = np.random.default_rng(1)
    eps = [([int(x) for x in rng.integers(0, 12, 3)], [(0, 5), (5, 10)]) for _ in range(300)]
    csr = csr_of(eps)
    ctx.load_arrays(types, times, 12)
    want = ctx.count_csr(csr).copy()
    p = tmp_path / "s.evt"
    write_events_binary(str(p), types, times, 12)
    ctx.load_file(str(p))
    assert np.array_equal(ctx.count_csr(csr), want)
    for t, tm, a, msg in (([0, 0], [5, 4], 1, "non-decreasing"), ([0, 0], [1, -4], 1, "negative event time"),
                          ([0, 3], [1, 4], 2, "type id out of range")):
        write_events_binary(str(p), np.array(t, np.uint32), np.array(tm, np.int64), a)
        with pytest.raises(DataError, match=msg):
            ctx.load_file(str(p))
    with pytest.raises(DataError, match="cannot open event file"):
        ctx.load_file(str(tmp_path / "missing.evt"))


def test_errors(ctx):
    with pytest.raises(DataError, match="non-decreasing"):
        ctx.load_arrays(np.array([0, 0], np.uint32), np.array([5, 4], np.int64), 1)
    with pytest.raises(DataError, match="negative event time"):
        ctx.load_arrays(np.array([0, 0], np.uint32), np.array([1, -4], np.int64), 1)
    with pytest.raises(DataError, match="type id out of range"):
        ctx.load_arrays(np.array([0, 3], np.uint32), np.array([1, 4], np.int64), 2)
    # first offending event decides
    with pytest.raises(DataError, match="type id out of range"):
        ctx.load_arrays(np.array([5, 0, 0], np.uint32), np.array([1, 0, -1], np.int64), 2)
    ctx.load_arrays(np.array([0, 1], np.uint32), np.array([0, 7], np.int64), 2)
    with pytest.raises(InvalidArgument, match="0 <= low < high"):
        ctx.count_csr(csr_of([([0, 1], [(5, 5)])]))
    with pytest.raises(InvalidArgument, match="at least one node"):
        ctx.count_csr(csr_of([([], [])]))
    with pytest.raises(Unsupported):
        ctx.count_csr(csr_of([([0, 1], [(5, 5000)])]))


@pytest.mark.parametrize("seed,high_max,gap_max", [(0, 250, 40), (1, 250, 400), (2, 4095, 900),
                                                   (3, 120, 10)])
def test_random_wide_windows_vs_port(ctx, seed, high_max, gap_max, segments_env):
    """Constraints with high > 63 take the wide-window kernels (local-memory
    history ring, bitmap rebuilt with a larger gap-compression cap)."""
    rng = np.random.default_rng(5000 + seed)
    for it in range(25):
        segments_env([None, 2, 5][it % 3])
        types, times, a, eps = _random_case(rng, 2500, 6, gap_max, 6, high_max)
        got = count_one(ctx, types, times, a, eps)
        csr = csr_of(eps)
        want = oracle.count_batch(types, times, csr.offsets, csr.types, csr.low, csr.high, threads=4)
        np.testing.assert_array_equal(got, want, err_msg=f"seed {seed} it {it}")
        # mixing back to a narrow batch on the same (rebuilt) bitmap stays exact
        narrow = [(t, [(lo % 40, min(hi, 63)) if lo % 40 < min(hi, 63) else (0, 5) for lo, hi in c])
                  for t, c in eps]
        got2 = ctx.count_csr(csr_of(narrow))
        csr2 = csr_of(narrow)
        want2 = oracle.count_batch(types, times, csr2.offsets, csr2.types, csr2.low, csr2.high, threads=4)
        np.testing.assert_array_equal(got2, want2, err_msg=f"narrow seed {seed} it {it}")


def _gen(name):
    if name == "cfg1":
        return GenConfig(26, 60, 32, [Embedding(Episode([0, 1, 2, 3], [(5, 10)] * 3), 2.0)], 1)
    if name == "cfg2":
        eps = [([0, 1, 2, 3], [BINS[1]] * 3), ([4, 5, 6, 7], [BINS[0], BINS[1], BINS[2]]),
               ([8, 9, 10, 11], [BINS[2], BINS[0], BINS[1]]), ([12, 13, 14, 15], [BINS[1], BINS[2], BINS[0]])]
        return GenConfig(26, 60, 32, [Embedding(Episode(t, c), 5.0) for t, c in eps], 1)
    if name == "cfg3":
        return GenConfig(64, 7813, 20, [], 3)
    raise KeyError(name)


def test_cfg1_all_pairs(ctx, golden_configs):
    g = golden_configs["cfg1"]
    types, times = generate_arrays(_gen("cfg1"))
    assert len(types) == g["n"]
    ctx.load_arrays(types, times, 26)
    eps = [([a, b], [(5, 10)]) for a in range(26) for b in range(26)]
    got = ctx.count_csr(csr_of(eps))
    assert [int(x) for x in got] == g["counts"]
    assert int(got.sum()) == g["sum"] == 176437
    assert fnv_u64s(got) == g["fnv_counts"]


@pytest.mark.parametrize("mode,knob", [(MODE_MINE, None), (MODE_EXACT, None), (MODE_MINE, "EPI_COMPACT_CUB"),
                                       (MODE_MINE, "EPI_PASS1_HULL"), (MODE_MINE, "EPI_WALK_SEQ"),
                                       (MODE_MINE, "EPI_MATERIALISE"), (MODE_MINE, "EPI_SURV_TC")])
def test_cfg2_mining(ctx, golden_configs, mode, knob, monkeypatch):
    """cfg2 mining CSV == the reference's, on the default device path and on
    each alternative it keeps (CUB multi-kernel compaction, hull pass 1,
    sequential concat walk, materialised candidates, multi-CTA survivor
    compaction)."""
    from paper_0905_2203_b200 import MiningConfig, mine, write_mining_csv, EventStream
    if knob:
        monkeypatch.setenv(knob, "1")
    g = golden_configs["cfg2"]
    types, times = generate_arrays(_gen("cfg2"))
    s = EventStream(types, times, 26)
    r = mine(s, MiningConfig(threshold=250, constraint_alphabet=BINS, max_level=4, mode=mode), ctx=ctx)
    assert [lv.candidates for lv in r.levels] == g["level_candidates"] == [26, 2028, 142228, 4]
    assert write_mining_csv(r) == g["csv"]
    if mode == MODE_MINE:
        assert r.stats["pruned"] > 0


@pytest.mark.parametrize("mode", [MODE_MINE, MODE_EXACT])
def test_mine_known_answers(ctx, golden_kats, mode):
    """T/test_miner.cpp mining cases (two-event stream, backend identity on
    random_stream(rng(82)), apriori closure on rng(81)): CSV and per-level
    candidate counts equal the reference's."""
    from paper_0905_2203_b200 import EventStream, MiningConfig, mine, write_mining_csv
    for k in golden_kats["mine"]:
        types, times, a = stream_from_json(k)
        s = EventStream(types, times, a)
        cfg = MiningConfig(threshold=k["threshold"], constraint_alphabet=[tuple(b) for b in k["alphabet_bins"]],
                           max_level=k["max_level"], mode=mode)
        r = mine(s, cfg, ctx=ctx)
        assert [lv.candidates for lv in r.levels] == k["level_candidates"], k["name"]
        assert write_mining_csv(r) == k["csv"], k["name"]


@pytest.mark.skipif(not oracle.ref_available(), reason="reference build (oracle/_ref) absent")
@pytest.mark.parametrize("seed", range(4))
def test_mine_random_vs_reference(ctx, seed):
    """Device-resident mining (both modes) == the reference's mine() run
    live (oracle/_ref) on random bursty streams: per-level candidate counts
    and the full CSV (episodes, order, counts)."""
    from paper_0905_2203_b200 import EventStream, MiningConfig, mine, write_mining_csv
    rng = np.random.default_rng(900 + seed)
    a = int(rng.integers(3, 9))
    n = int(rng.integers(2000, 6000))
    times = np.cumsum(rng.integers(0, [2, 4, 8, 16][seed] + 1, n)).astype(np.int64)
    types = rng.integers(0, a, n).astype(np.uint32)
    bins = [[(0, 5), (5, 10), (10, 15)], [(0, 4), (2, 7)], [(1, 9)], [(0, 3), (3, 6), (6, 9), (9, 12)]][seed]
    thr = int(max(2, n // (a * a * 4)))
    csv_ref, cands_ref, _ = oracle.ref_mine(types, times, a, thr, bins, 5, switch_level=99, backend=0,
                                            workers=4)
    s = EventStream(types, times, a)
    for mode in (MODE_MINE, MODE_EXACT):
        r = mine(s, MiningConfig(threshold=thr, constraint_alphabet=bins, max_level=5, mode=mode), ctx=ctx)
        assert [lv.candidates for lv in r.levels] == cands_ref, (seed, mode)
        assert write_mining_csv(r) == csv_ref, (seed, mode)


def test_mine_acceptance_c3(ctx):
    """T/acceptance.cpp C3: four 9-node chains embedded at 1 Hz in 100 s of
    64-neuron 20 Hz noise are all frequent at level 9 (threshold 50)."""
    from paper_0905_2203_b200 import EventStream, MiningConfig, mine
    chains = [Episode(list(range(9 * e, 9 * e + 9)), [(5, 10)] * 8) for e in range(4)]
    types, times = generate_arrays(GenConfig(64, 100, 20, [Embedding(c, 1.0) for c in chains], 99177))
    r = mine(EventStream(types, times, 64), MiningConfig(threshold=50, constraint_alphabet=[(5, 10)],
                                                           max_level=9), ctx=ctx)
    assert len(r.levels) >= 9 and r.levels[8].level == 9
    found = {tuple(ep.types) for ep, _ in r.levels[8].frequent}
    assert all(tuple(c.types) in found for c in chains)


def test_cfg2_level3_bounds_sound(ctx, golden_configs):
    """Pass 1 never prunes a frequent candidate, and its bound is >= exact."""
    from paper_0905_2203_b200 import generate_candidates, Episode as E
    types, times = generate_arrays(_gen("cfg2"))
    ctx.load_arrays(types, times, 26)
    l1 = [E([t], []) for t in range(26)]
    l2 = generate_candidates(2, l1, BINS, 26)
    c2 = ctx.count_csr(csr_of([(e.types, e.constraints) for e in l2]))
    f2 = [e for e, c in zip(l2, c2) if c >= 250]
    l3 = generate_candidates(3, f2, BINS, 26)
    assert len(l3) == 142228
    csr3 = csr_of([(e.types, e.constraints) for e in l3])
    exact = ctx.count_csr(csr3, threshold=250, mode=MODE_EXACT)
    mined, freq = ctx.count_csr(csr3, threshold=250, mode=MODE_MINE, with_frequent=True)
    keep = mined != np.uint64(COUNT_PRUNED)
    np.testing.assert_array_equal(mined[keep], exact[keep])
    assert np.all(exact[~keep] < 250)
    np.testing.assert_array_equal(freq.astype(bool), exact >= 250)
    assert int((exact >= 250).sum()) == 8


def test_cfg3_first_candidates(ctx, golden_configs):
    g = golden_configs["cfg3"]
    types, times = generate_arrays(_gen("cfg3"))
    assert len(types) == g["n"] == 10004428
    ctx.load_arrays(types, times, 64)
    eps = [ep_from_json(e) for e in g["episodes"]]
    got = ctx.count_csr(csr_of(eps))
    assert [int(x) for x in got] == g["counts"]
    assert int(got[:64].sum()) == g["sum_first64"] == 87180


@pytest.mark.parametrize("alphabet", [300, 1000, 4000])
def test_large_alphabets(ctx, alphabet):
    """Bitmap blocks beyond the shared-memory ring (alphabet > ~340 types read
    rows from global memory) and the spare zero row."""
    rng = np.random.default_rng(alphabet)
    n = 60000
    times = np.cumsum(rng.integers(0, 3, n)).astype(np.int64)
    hot = rng.integers(0, 20, n)          # a few frequent types so counts are non-zero
    types = np.where(rng.random(n) < 0.7, hot, rng.integers(0, alphabet, n)).astype(np.uint32)
    eps = [([int(a), int(b), int(c)], [(0, 5), (2, 9)]) for a, b, c in rng.integers(0, 20, (150, 3))]
    eps += [([int(a), int(b)], [(1, 30)]) for a, b in rng.integers(0, alphabet, (100, 2))]
    got = count_one(ctx, types, times, alphabet, eps)
    csr = csr_of(eps)
    want = oracle.count_batch(types, times, csr.offsets, csr.types, csr.low, csr.high, threads=8)
    np.testing.assert_array_equal(got, want)
    assert int(got.sum()) > 0


def test_million_candidates(ctx):
    """10^6 candidates in one batch (cfg5's largest candidate set) on a 1M
    event stream: seeded subset against the oracle."""
    rng = np.random.default_rng(7)
    types, times = generate_arrays(GenConfig(64, 1_000_000 / (64 * 20), 20, [], 77))
    ctx.load_arrays(types, times, 64)
    m = 1_000_000
    t = rng.integers(0, 64, (m, 3)).astype(np.uint32)
    b = rng.integers(0, 3, (m, 2))
    lo = np.array([0, 5, 10], np.int64)[b].reshape(-1)
    from paper_0905_2203_b200 import CSR
    csr = CSR(np.arange(0, 3 * m + 1, 3, dtype=np.uint32), t.reshape(-1), lo, lo + 5)
    got = ctx.count_csr(csr)
    pick = np.sort(rng.choice(m, 64, replace=False))
    sub = csr_of([([int(x) for x in t[i]], [(int(lo[2 * i]), int(lo[2 * i]) + 5),
                                            (int(lo[2 * i + 1]), int(lo[2 * i + 1]) + 5)]) for i in pick])
    want = oracle.count_batch(types, times, sub.offsets, sub.types, sub.low, sub.high, threads=16)
    np.testing.assert_array_equal(got[pick], want)


@pytest.mark.parametrize("seed", range(4))
def test_uniform_head_last_width_vs_port(ctx, seed, segments_env):
    """Batches whose constraints before the last share one width W and whose
    last constraints share another width WL (the shape of the miner's pass-1
    hull episodes) take the launch_machines_last kernels; every high <= 32."""
    rng = np.random.default_rng(7000 + seed)
    for it in range(24):
        segments_env([None, 4, 9][it % 3])
        n_types = int(rng.integers(3, 9))
        n_ev = 3000
        times = np.cumsum(rng.integers(0, [3, 12, 60][it % 3] + 1, n_ev)).astype(np.int64)
        types = rng.integers(0, n_types, n_ev).astype(np.uint32)
        W = int(rng.integers(1, 17))
        WL = int(rng.integers(1, 17))
        eps = []
        for _ in range(int(rng.integers(40, 300))):
            N = int(rng.integers(3, 7))
            cons = []
            for k in range(N - 1):
                w = W if k + 1 < N - 1 else WL
                lo = int(rng.integers(0, 32 - w + 1))
                cons.append((lo, lo + w))
            eps.append(([int(x) for x in rng.integers(0, n_types, N)], cons))
        # one length per batch keeps the launch on a single specialised kernel
        N0 = len(eps[0][0])
        eps = [e for e in eps if len(e[0]) == N0]
        got = count_one(ctx, types, times, n_types, eps)
        csr = csr_of(eps)
        want = oracle.count_batch(types, times, csr.offsets, csr.types, csr.low, csr.high, threads=4)
        np.testing.assert_array_equal(got, want, err_msg=f"seed {seed} it {it} W {W} WL {WL}")


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("pass1", ["popcount", "hull"])
def test_mine_pass1_every_level_vs_reference(ctx, seed, pass1, monkeypatch):
    """Pass 1 forced onto every level >= 2 (EPI_PASS1_MIN=1), with the
    popcount bound (default) or the hull relaxation (EPI_PASS1_HULL): the
    mining CSV must still equal the reference's mine() (no frequent episode
    pruned, survivors' counts exact), up to level 5 and over several
    constraint alphabets (mixed widths, lo > 0)."""
    from paper_0905_2203_b200 import EventStream, MiningConfig, mine, write_mining_csv
    monkeypatch.setenv("EPI_PASS1_MIN", "1")
    if pass1 == "hull":
        monkeypatch.setenv("EPI_PASS1_HULL", "1")
    rng = np.random.default_rng(4200 + seed)
    a = int(rng.integers(3, 8))
    n = int(rng.integers(2000, 5000))
    times = np.cumsum(rng.integers(0, [2, 4, 8, 3, 6, 12][seed] + 1, n)).astype(np.int64)
    types = rng.integers(0, a, n).astype(np.uint32)
    bins = [[(0, 5), (5, 10), (10, 15)], [(0, 4), (2, 7)], [(1, 9)], [(0, 3), (3, 6), (6, 9), (9, 12)],
            [(0, 10), (10, 32)], [(4, 6), (0, 2), (20, 31)]][seed]
    thr = int(max(2, n // (a * a * 3)))
    csv_ref, cands_ref, _ = oracle.ref_mine(types, times, a, thr, bins, 5, switch_level=99, backend=0,
                                            workers=4)
    s = EventStream(types, times, a)
    r = mine(s, MiningConfig(threshold=thr, constraint_alphabet=bins, max_level=5, mode=MODE_MINE), ctx=ctx)
    assert [lv.candidates for lv in r.levels] == cands_ref, seed
    assert write_mining_csv(r) == csv_ref, seed


@pytest.mark.parametrize("seed", range(3))
def test_mine_wide_windows_vs_reference(ctx, seed, monkeypatch):
    """Constraint alphabets with high > 32 (popcount pass 1 off; the
    last-constraint hull pass 1 forced on every level; wide-window map
    kernels for high > 63): mining CSV == the reference's mine()."""
    from paper_0905_2203_b200 import EventStream, MiningConfig, mine, write_mining_csv
    monkeypatch.setenv("EPI_PASS1_MIN", "1")
    rng = np.random.default_rng(5100 + seed)
    a = int(rng.integers(3, 6))
    n = int(rng.integers(1500, 3000))
    times = np.cumsum(rng.integers(0, [20, 40, 10][seed] + 1, n)).astype(np.int64)
    types = rng.integers(0, a, n).astype(np.uint32)
    bins = [[(0, 40), (40, 80)], [(10, 50), (0, 120)], [(0, 33), (33, 66), (66, 99)]][seed]
    thr = int(max(2, n // (a * a * 2)))
    csv_ref, cands_ref, _ = oracle.ref_mine(types, times, a, thr, bins, 4, switch_level=99, backend=0,
                                            workers=4)
    s = EventStream(types, times, a)
    for mode in (MODE_MINE, MODE_EXACT):
        r = mine(s, MiningConfig(threshold=thr, constraint_alphabet=bins, max_level=4, mode=mode), ctx=ctx)
        assert [lv.candidates for lv in r.levels] == cands_ref, (seed, mode)
        assert write_mining_csv(r) == csv_ref, (seed, mode)


def test_mine_stats_stable_across_graph_replays(ctx, monkeypatch):
    """The statistics a mining call reports (device counters resolved from the
    log, event timings resolved while the next level runs) are the same for a
    direct run, the captured run and graph replays."""
    types, times = generate_arrays(_gen("cfg2"))
    ctx.load_arrays(types, times, 26)
    keys = ("episodes", "pass1_groups", "pass2_episodes", "pruned", "segments", "patches",
            "episode_events", "tile_steps", "bound_words")
    monkeypatch.setenv("EPI_NO_GRAPH", "1")
    want = ctx.mine_raw(250, BINS, 4, MODE_MINE)[5]
    monkeypatch.delenv("EPI_NO_GRAPH")
    for it in range(4):
        st = ctx.mine_raw(250, BINS, 4, MODE_MINE)[5]
        assert {k: st[k] for k in keys} == {k: want[k] for k in keys}, it
        assert st["bound_ms"] > 0 and st["pass2_ms"] > 0, it
        assert abs(st["pass1_ms"] + st["pass2_ms"] - st["total_ms"]) < 1e-3, it
        assert st["map_ms"] + st["concat_ms"] <= st["pass2_ms"] + 1e-3, it


def test_mine_graph_replay(ctx, golden_configs, monkeypatch):
    """Per-level CUDA graphs: repeated mining of cfg2 (first run direct,
    second captured, then replayed) and, interleaved, of a type-relabelled
    copy of the stream whose levels have the same sizes (so the same graph
    keys replay with other data): every run's CSV equals the graph-free
    result, and the original's equals the reference's."""
    from paper_0905_2203_b200 import EventStream, MiningConfig, mine, write_mining_csv
    g = golden_configs["cfg2"]
    types, times = generate_arrays(_gen("cfg2"))
    perm = np.random.default_rng(8).permutation(26).astype(np.uint32)
    relabeled = perm[types]
    cfg = MiningConfig(threshold=250, constraint_alphabet=BINS, max_level=4, mode=MODE_MINE)
    monkeypatch.setenv("EPI_NO_GRAPH", "1")
    ref_rel = mine(EventStream(relabeled, times, 26), cfg, ctx=ctx)
    want_rel = write_mining_csv(ref_rel)
    monkeypatch.delenv("EPI_NO_GRAPH")
    for it in range(4):
        r = mine(EventStream(types, times, 26), cfg, ctx=ctx)
        assert write_mining_csv(r) == g["csv"], it
        assert [lv.candidates for lv in r.levels] == g["level_candidates"]
        r2 = mine(EventStream(relabeled, times, 26), cfg, ctx=ctx)
        assert write_mining_csv(r2) == want_rel, it
        # statistics replayed with the graph equal the graph-free run's
        for key in ("pruned", "pass2_episodes", "episodes"):
            assert r2.stats[key] == ref_rel.stats[key], (it, key)


@pytest.mark.parametrize("case", ["narrow", "wide_types", "wide_gaps", "huge_gaps"])
def test_encoded_ingest_matches_raw(ctx, case, monkeypatch):
    """Streams of >= 4M events cross PCIe encoded (ingest.cu: narrowed types,
    per-event time deltas against a base every 2048 events); the device SoA
    they decode to must give the counts of the raw 12 B/event upload."""
    rng = np.random.default_rng(["narrow", "wide_types", "wide_gaps", "huge_gaps"].index(case))
    n = 5_000_000
    a = 300 if case == "wide_types" else 40
    gmax = {"narrow": 4, "wide_types": 4, "wide_gaps": 5000, "huge_gaps": 1 << 40}[case]
    gaps = rng.integers(0, 4, n)
    jumps = rng.random(n) < 1e-4
    gaps[jumps] = rng.integers(0, gmax, int(jumps.sum()), dtype=np.int64) if gmax > 4 else gaps[jumps]
    times = np.cumsum(gaps).astype(np.int64)
    types = rng.integers(0, a, n).astype(np.uint32)
    eps = [([int(x) for x in rng.integers(0, a, 3)], [BINS[int(b)] for b in rng.integers(0, 3, 2)])
           for _ in range(300)]
    csr = csr_of(eps)
    ctx.load_arrays(types, times, a)
    got = ctx.count_csr(csr)
    monkeypatch.setenv("EPI_RAW_INGEST", "1")
    ctx.load_arrays(types, times, a)
    np.testing.assert_array_equal(got, ctx.count_csr(csr))


@pytest.mark.parametrize("where", [0, 2047, 2048, 262144, 4_999_999])
def test_encoded_ingest_reports_first_offender(ctx, where):
    """A chunk holding an invalid event ships raw, so the device validation
    reports the reference's message (E/types.hpp:109-111) on the encoded path
    as on the raw one."""
    n = 5_000_000
    types = (np.arange(n) % 7).astype(np.uint32)
    times = np.arange(n, dtype=np.int64)
    for kind in ("regress", "negative", "type"):
        t, tm = types.copy(), times.copy()
        if kind == "regress" and where > 0:
            tm[where] = tm[where - 1] - 1
        elif kind == "negative" or (kind == "regress" and where == 0):
            tm[: where + 1] -= where + 5
        else:
            t[where] = 9
        want = {"regress": "non-decreasing", "negative": "negative event time", "type": "out of range"}[kind]
        with pytest.raises(DataError, match=want if not (kind == "regress" and where == 0) else "negative"):
            ctx.load_arrays(t, tm, 7)
