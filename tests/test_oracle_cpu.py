"""The CPU checker itself, pinned before it is trusted: the oracle port
(oracle/episodic_oracle.c) against the reference's known-answer tests and
randomised corpora recorded from the reference (tests/golden/), and - when
the reference build (oracle/_ref) is present - against the reference run
live on fresh instances."""
import numpy as np
import pytest

import oracle
from helpers import ep_from_json, stream_from_json
from instances import corpus, fnv_stream


def _cons(cons):
    return [c[0] for c in cons], [c[1] for c in cons]


def test_port_known_answer_tests(golden_kats):
    for k in golden_kats["count"]:
        types, times, a = stream_from_json(k)
        et, cons = ep_from_json(k["episode"])
        lo, hi = _cons(cons)
        assert oracle.count_fsm(types, times, et, lo, hi) == k["expected"] == k["count_fsm"], k["name"]
        if len(types) <= 500:
            assert oracle.oracle_count(types, times, et, lo, hi) == k["expected"], k["name"]


def test_instance_rng_restatement_matches_reference(golden_instances):
    """tests/instances.py regenerates the reference's InstanceRng streams
    bit-exactly (FNV digest per stream recorded from the reference)."""
    for c in golden_instances:
        gen = corpus(c["seed"], c["count"], c["max_events"], c["max_alphabet"], c["max_gap"], c["max_size"])
        for (types, times, a, et, cons), want in zip(gen, c["instances"]):
            assert fnv_stream(types, times, a) == want["fnv"]
            assert et == want["episode"]["types"]
            assert [list(x) for x in cons] == want["episode"]["constraints"]


def test_port_equals_reference_on_corpora(golden_instances):
    """count_fsm and oracle_count restated == the reference's count_fsm on
    all 2,250 instances of T/test_fsm.cpp, T/test_tracking.cpp,
    T/test_mapconcat.cpp and acceptance C1."""
    n = 0
    for c in golden_instances:
        gen = corpus(c["seed"], c["count"], c["max_events"], c["max_alphabet"], c["max_gap"], c["max_size"])
        for (types, times, a, et, cons), want in zip(gen, c["instances"]):
            lo, hi = _cons(cons)
            assert oracle.count_fsm(types, times, et, lo, hi) == want["count"]
            assert oracle.oracle_count(types, times, et, lo, hi) == want["count"]
            n += 1
    assert n == 2250


def test_max_nonoverlap_hand_traces():
    """T/test_oracle.cpp:82-91."""
    assert oracle.max_nonoverlap([]) == 0
    assert oracle.max_nonoverlap([(1, 3), (2, 4), (5, 6)]) == 2
    assert oracle.max_nonoverlap([(0, 5)]) == 1
    assert oracle.max_nonoverlap([(5, 5), (5, 5)]) == 1
    assert oracle.max_nonoverlap([(5, 5), (6, 6)]) == 2
    assert oracle.max_nonoverlap([(0, 3), (3, 6)]) == 1


def test_max_nonoverlap_vs_brute_force():
    """T/test_oracle.cpp:93-105 shape: greedy == exhaustive subset search."""
    from itertools import combinations
    rng = np.random.default_rng(43)
    for _ in range(150):
        k = int(rng.integers(0, 9))
        occ = []
        for _ in range(k):
            a = int(rng.integers(0, 31))
            occ.append((a, a + int(rng.integers(0, 11))))
        best = 0
        for r in range(len(occ) + 1):
            for sub in combinations(sorted(occ), r):
                if all(sub[i][0] > sub[i - 1][1] for i in range(1, len(sub))):
                    best = max(best, r)
        assert oracle.max_nonoverlap(occ) == best


def test_validation_messages():
    assert oracle.validate_stream([0, 0], [5, 4], 1) == (2, "event times must be non-decreasing")
    assert oracle.validate_stream([0], [-1], 1) == (2, "negative event time")
    assert oracle.validate_stream([0, 3], [1, 4], 2) == (2, "event type id out of range")
    assert oracle.validate_stream([0, 1], [1, 4], 2) == (0, "")


def test_port_batch_threads_deterministic():
    rng = np.random.default_rng(7)
    times = np.cumsum(rng.integers(0, 4, 3000)).astype(np.int64)
    types = rng.integers(0, 5, 3000).astype(np.uint32)
    eps = [([int(x) for x in rng.integers(0, 5, 3)], [(0, 5), (5, 10)]) for _ in range(50)]
    off = np.cumsum([0] + [3] * 50).astype(np.uint32)
    et = np.array([t for e, _ in eps for t in e], np.uint32)
    lo = np.array([c[0] for _, cs in eps for c in cs], np.int64)
    hi = np.array([c[1] for _, cs in eps for c in cs], np.int64)
    a = oracle.count_batch(types, times, off, et, lo, hi, threads=1)
    b = oracle.count_batch(types, times, off, et, lo, hi, threads=8)
    np.testing.assert_array_equal(a, b)


@pytest.mark.skipif(not oracle.ref_available(), reason="reference build (oracle/_ref) absent")
def test_port_equals_live_reference_on_fresh_instances():
    """Fresh random instances (not in the fixtures): port == reference
    count_fsm == reference count_tracking == reference count_mapconcat."""
    rng = np.random.default_rng(2024)
    for it in range(40):
        n = int(rng.integers(0, 800))
        a = int(rng.integers(1, 7))
        times = np.cumsum(rng.integers(0, [3, 9, 40][it % 3] + 1, n)).astype(np.int64)
        types = rng.integers(0, a, n).astype(np.uint32)
        eps = []
        for _ in range(20):
            N = int(rng.integers(1, 6))
            cons = []
            for _k in range(N - 1):
                h = int(rng.integers(1, 64))
                cons.append((int(rng.integers(0, h)), h))
            eps.append(([int(x) for x in rng.integers(0, a, N)], cons))
        off = np.cumsum([0] + [len(t) for t, _ in eps]).astype(np.uint32)
        et = np.array([t for e, _ in eps for t in e], np.uint32)
        lo = np.array([c[0] for _, cs in eps for c in cs], np.int64)
        hi = np.array([c[1] for _, cs in eps for c in cs], np.int64)
        port = oracle.count_batch(types, times, off, et, lo, hi)
        for algo in ("fsm", "tracking", "mapconcat"):
            ref = oracle.ref_count_batch(types, times, a, off, et, lo, hi, algo=algo, workers=2)
            np.testing.assert_array_equal(port, ref, err_msg=f"{algo} it {it}")


def test_scale_fixture_agrees_with_config_fixture(golden_configs):
    """tests/golden/scale.json (reference, all 10,000 cfg3 candidates) and
    configs.json (reference, first 256) were written by separate runs."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "scale.json")) as f:
        scale = json.load(f)
    assert scale["cfg3"]["counts"][:256] == golden_configs["cfg3"]["counts"]
    assert scale["cfg3"]["n"] == golden_configs["cfg3"]["n"]
    assert len(scale["cfg3"]["counts"]) == 10000
    for name, cell in scale.items():
        assert len(cell["counts"]) >= 1000, name
        assert sum(cell["counts"]) == cell["sum"], name
