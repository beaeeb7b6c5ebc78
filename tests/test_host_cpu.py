"""Host-side pieces that need no GPU: the C-ABI library loads and exports
every symbol include/episodic_b200.h declares; the host Apriori join and
the synthetic generator equal the reference's (golden fixtures); the Python
mirror's validation and formatting; no silent CPU fallback."""
import os
import re

import numpy as np
import pytest

import oracle
from conftest import ROOT
from helpers import ep_from_json
from paper_0905_2203_b200 import (DataError, Embedding, Episode, EpisodicError, EventStream, GenConfig,
                                  InvalidArgument, LevelResult, MiningResult, _native, format_episode,
                                  generate_arrays, generate_candidates, write_mining_csv)


def test_library_exports_every_declared_symbol():
    with open(os.path.join(ROOT, "include", "episodic_b200.h")) as f:
        header = f.read()
    declared = set(re.findall(r"^\s*(?:const char\*|epi_status|void|uint64_t|uint32_t|int)\s+(epi_\w+)\(", header,
                              re.M))
    assert "epi_count" in declared and "epi_mine" in declared and len(declared) >= 12
    for name in declared:
        assert hasattr(_native.lib, name), name
    assert set(_native.EXPORTS) == declared


def test_library_is_sm100a():
    so = _native.LIB_PATH
    out = os.popen(f"cuobjdump -lelf {so} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_no_device_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_0905_2203_b200 import Context
    with pytest.raises(EpisodicError):
        Context(0)


def _ep(j):
    t, c = ep_from_json(j)
    return Episode(t, c)


def test_generate_candidates_known_answers(golden_kats):
    """Join of E/miner.hpp:76-109 (order included) == the reference's on the
    T/test_miner.cpp KATs plus repeated-type and level-2 cases."""
    for k in golden_kats["candidates"]:
        freq = [_ep(f) for f in k["frequent"]]
        got = generate_candidates(k["level"], freq, [tuple(b) for b in k["alphabet_bins"]], k["alphabet"])
        want = [_ep(c) for c in k["candidates"]]
        assert got == want, k["name"]


def test_generate_candidates_cfg2_level3(golden_configs):
    g = golden_configs["cfg2"]
    lvl2 = []
    for line in g["csv"].splitlines()[1:]:
        lv, ep, _ = line.split(",")[0], ",".join(line.split(",")[1:-1]), line.split(",")[-1]
        if lv == "2":
            parts = ep.split("-")
            lo, hi = parts[1][1:-1].split(",")
            lvl2.append(Episode([int(parts[0]), int(parts[2])], [(int(lo), int(hi))]))
    assert len(lvl2) == 1917
    c3 = generate_candidates(3, lvl2, [(0, 5), (5, 10), (10, 15)], 26)
    assert len(c3) == g["level_candidates"][2] == 142228


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "acceptance_c2", "datagen_injections",
                                  "datagen_reproducible", "cfg3"])
def test_generator_matches_reference(golden_datagen, name):
    """epi_generate restates generate() (E/datagen.hpp:71-122) bit-exactly."""
    bins = [(0, 5), (5, 10), (10, 15)]
    cfgs = {
        "cfg1": GenConfig(26, 60, 32, [Embedding(Episode([0, 1, 2, 3], [(5, 10)] * 3), 2.0)], 1),
        "cfg2": GenConfig(26, 60, 32, [Embedding(Episode(t, c), 5.0) for t, c in [
            ([0, 1, 2, 3], [bins[1]] * 3), ([4, 5, 6, 7], [bins[0], bins[1], bins[2]]),
            ([8, 9, 10, 11], [bins[2], bins[0], bins[1]]), ([12, 13, 14, 15], [bins[1], bins[2], bins[0]])]], 1),
        "acceptance_c2": GenConfig(64, 100, 20, [Embedding(Episode([0, 1, 2, 3, 4], [(5, 10)] * 4), 1.0)], 424242),
        "datagen_injections": GenConfig(8, 20, 10, [Embedding(Episode([0, 1, 2, 3], [(5, 10), (5, 10), (0, 6)]),
                                                               2.0)], 17),
        "datagen_reproducible": GenConfig(1, 1_000_000, 1.0, [], 99),
        "cfg3": GenConfig(64, 7813, 20, [], 3),
    }
    want = next(d for d in golden_datagen if d["name"] == name)
    cfg = cfgs[name]
    types, times = generate_arrays(cfg)
    assert len(types) == want["n"]
    assert oracle.fnv_stream(types, times, cfg.neurons) == want["fnv"]


def test_generator_rejects_invalid_configs():
    """T/test_datagen.cpp:92-100 and E/datagen.hpp:72-80 messages."""
    with pytest.raises(InvalidArgument, match="base rate"):
        generate_arrays(GenConfig(base_rate_hz=0))
    with pytest.raises(InvalidArgument, match="unknown neuron"):
        generate_arrays(GenConfig(neurons=2, base_rate_hz=10,
                                  embedded=[Embedding(Episode([0, 5], [(5, 10)]), 1.0)]))
    with pytest.raises(InvalidArgument, match="at least one neuron"):
        generate_arrays(GenConfig(neurons=0))
    assert len(generate_arrays(GenConfig(duration_s=0))[0]) == 0


def test_generator_sorted_ties_by_neuron():
    types, times = generate_arrays(GenConfig(16, 30, 50, [], 5))
    assert np.all(np.diff(times) >= 0)
    tie = np.diff(times) == 0
    assert np.all(np.diff(types.astype(np.int64))[tie] >= 0)


def test_from_events_validation():
    with pytest.raises(DataError, match="non-decreasing"):
        EventStream.from_events([(0, 5), (0, 4)], 1)
    with pytest.raises(DataError, match="negative"):
        EventStream.from_events([(0, -1)], 1)
    with pytest.raises(DataError, match="out of range"):
        EventStream.from_events([(3, 1)], 2)
    s = EventStream.from_events([(0, 1), (1, 1), (0, 4)], 2)
    assert s.size() == 3 and s.alphabet_size() == 2 and s.time_at(2) == 4


def test_formatting_matches_reference_grammar():
    """format_episode (E/grammar.hpp:70-83) and write_mining_csv
    (E/miner.hpp:175-181): `2,0-(5,10]-1,1` (T/test_miner.cpp:134-151)."""
    ep = Episode([0, 1], [(5, 10)])
    assert format_episode(ep) == "0-(5,10]-1"
    r = MiningResult([LevelResult(1, 2, [(Episode([0], []), 1), (Episode([1], []), 1)]),
                      LevelResult(2, 4, [(ep, 1)])])
    csv = write_mining_csv(r)
    assert csv.startswith("level,episode,count\n") and "2,0-(5,10]-1,1" in csv


def test_generate_candidates_empty_and_level1():
    assert generate_candidates(2, [], [(5, 10)], 3) == []
    assert generate_candidates(5, [], [(5, 10)], 3) == []
    assert generate_candidates(1, [], [(5, 10)], 2) == [Episode([0], []), Episode([1], [])]


def test_reference_arm_loads_only_the_reference():
    """bench.py --impl reference runs the reference compiled in place
    (oracle/_ref) and nothing of this package: its JSON line lists the
    in-repo shared objects the process loaded."""
    import json
    import subprocess
    import sys
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    libs = line["native_so_loaded"]
    assert any("oracle/_ref" in p for p in libs), libs
    assert not any("paper_0905_2203_b200" in p for p in libs), libs


def test_reference_arm_candidates_equal_product_draws():
    """The reference arm's pure-Python candidate draws (oracle.mt_episodes)
    == this package's seeded generator (epi_random_episodes, host code)."""
    from paper_0905_2203_b200 import random_episodes_csr
    for seed, nodes, alphabet in ((55, 3, 64), (44, 5, 60), (5, 3, 64)):
        eps = oracle.mt_episodes(seed, 200, nodes, alphabet, [(0, 5), (5, 10), (10, 15)])
        csr = random_episodes_csr(seed, 200, nodes, alphabet, [(0, 5), (5, 10), (10, 15)])
        assert [csr.episode(i) for i in range(200)] == [(list(t), [tuple(c) for c in cs]) for t, cs in eps]


def test_bench_cpu_baseline_leg():
    """bench.py's cpu_baseline object (rank 0, N=1) on the cfg1 workload:
    the reference timed on host cores, with the fields the contract names."""
    import argparse
    import sys
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    sys.path.insert(0, ROOT)
    import bench
    types, times, alphabet = bench.make_stream("cfg1")
    args = argparse.Namespace(config="cfg1", cfg5_events=10_000_000, cfg5_cands=1_000_000)
    cb = bench.cpu_baseline_for(args, types, times, alphabet)
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] == "reference"
    assert "1 step(s)" in cb["sample"] and cb["unit"] == "episode-events/s"
