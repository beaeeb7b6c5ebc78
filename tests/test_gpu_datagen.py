"""Device generator (epi_generate_stream, gen_dev.cu) == the reference's
generate() (E/datagen.hpp:71-122) bit for bit: stream digests of the
reference-written fixtures (tests/golden/datagen.json, scale.json) and
element-wise equality with the host restatement on the bench configs."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_0905_2203_b200 import Context, Embedding, Episode, GenConfig, generate_arrays

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BINS = [(0, 5), (5, 10), (10, 15)]


def _gen_cfg(name):
    if name == "cfg1":
        return GenConfig(26, 60, 32, [Embedding(Episode([0, 1, 2, 3], [(5, 10)] * 3), 2.0)], 1)
    if name == "cfg2":
        eps = [([0, 1, 2, 3], [BINS[1]] * 3), ([4, 5, 6, 7], [BINS[0], BINS[1], BINS[2]]),
               ([8, 9, 10, 11], [BINS[2], BINS[0], BINS[1]]), ([12, 13, 14, 15], [BINS[1], BINS[2], BINS[0]])]
        return GenConfig(26, 60, 32, [Embedding(Episode(t, c), 5.0) for t, c in eps], 1)
    if name == "cfg3":
        return GenConfig(64, 7813, 20, [], 3)
    raise KeyError(name)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_device_generate_matches_reference_digest(ctx, name):
    want = {d["name"]: d for d in json.load(open(os.path.join(GOLDEN, "datagen.json")))}[name]
    ctx.generate(_gen_cfg(name))
    types, times = ctx.download()
    assert len(types) == want["n"]
    assert oracle.fnv_stream(types, times, _gen_cfg(name).neurons) == want["fnv"]
    ht, htm = generate_arrays(_gen_cfg(name))
    np.testing.assert_array_equal(types, ht)
    np.testing.assert_array_equal(times, htm)


def test_device_generate_fixture_configs(ctx):
    """The other generator configurations of the reference fixture
    (acceptance C2 with an embedded 5-chain, injections, a 1-neuron stream of
    1M seconds): digests equal."""
    want = {d["name"]: d for d in json.load(open(os.path.join(GOLDEN, "datagen.json")))}
    chain5 = Episode([0, 1, 2, 3, 4], [(5, 10)] * 4)
    cfgs = {"acceptance_c2": GenConfig(64, 100, 20, [Embedding(chain5, 1.0)], 424242),
            "datagen_injections": GenConfig(8, 20, 10, [Embedding(Episode([0, 1, 2, 3], [(5, 10), (5, 10), (0, 6)]),
                                                                  2.0)], 17),
            "datagen_reproducible": GenConfig(1, 1_000_000, 1.0, [], 99)}
    for name, cfg in cfgs.items():
        ctx.generate(cfg)
        types, times = ctx.download()
        assert len(types) == want[name]["n"], name
        assert oracle.fnv_stream(types, times, cfg.neurons) == want[name]["fnv"], name


@pytest.mark.parametrize("n", [1_000_000, 100_000_000, 1_000_000_000])
def test_device_generate_scale_streams(ctx, n):
    """cfg5 streams up to 1B events: digest of the reference generate()
    output (tests/golden/scale.json, written with oracle/_ref) and counts of
    the cell's reference-checked candidates on the device-generated stream."""
    scale = json.load(open(os.path.join(GOLDEN, "scale.json")))
    cell = scale[f"cfg5_{n}"]
    s = cell["stream"]
    ctx.generate(GenConfig(s["neurons"], s["duration_s"], s["rate_hz"], [], s["seed"]))
    types, times = ctx.download()
    assert len(types) == cell["n"]
    assert oracle.fnv_stream(types, times, 64) == cell["stream_fnv"]
    from paper_0905_2203_b200 import random_episodes_csr
    c = cell["cands"]
    got = ctx.count_csr(random_episodes_csr(c["seed"], c["count"], c["nodes"], c["alphabet"], BINS))
    np.testing.assert_array_equal(got, np.array(cell["counts"], np.uint64))


def test_device_generate_errors(ctx):
    from paper_0905_2203_b200 import InvalidArgument
    with pytest.raises(InvalidArgument, match="at least one neuron"):
        ctx.generate(GenConfig(0, 10, 20, [], 1))
    with pytest.raises(InvalidArgument, match="base rate"):
        ctx.generate(GenConfig(4, 10, 0, [], 1))
    with pytest.raises(InvalidArgument, match="unknown neuron"):
        ctx.generate(GenConfig(4, 10, 20, [Embedding(Episode([0, 9], [(0, 5)]), 1.0)], 1))


@pytest.mark.parametrize("cfg", [
    dict(electrodes=12, duration_s=300, seed=7),
    dict(electrodes=5, duration_s=50, seed=9, burst_gain=1.0),
    dict(electrodes=7, duration_s=80, seed=11, burst_rate_hz=0.0),
    dict(electrodes=9, duration_s=120, seed=13, burst_rate_hz=2.0, burst_min_ms=5, burst_max_ms=40),
])
def test_device_bursty_equals_host(ctx, cfg):
    """epi_generate_bursty_stream == the host bursty generator (element-wise),
    with and without bursts, extra rate 0, short dense bursts, embedded
    episodes."""
    from paper_0905_2203_b200 import BurstConfig, generate_bursty_arrays
    bc = BurstConfig(embedded=[Embedding(Episode([0, 1, 2], [(5, 10), (0, 5)]), 0.7)], **cfg)
    ht, htm = generate_bursty_arrays(bc)
    ctx.generate_bursty(bc)
    types, times = ctx.download()
    np.testing.assert_array_equal(types, ht)
    np.testing.assert_array_equal(times, htm)


def test_device_bursty_cfg4_matches_fixture(ctx):
    """cfg4's ~100M-event stream generated on the device: the digest the
    reference-checked scale fixture was computed on."""
    from paper_0905_2203_b200 import BurstConfig
    cell = json.load(open(os.path.join(GOLDEN, "scale.json")))["cfg4"]
    s = cell["stream"]
    emb = [Embedding(Episode(t, [tuple(c) for c in cs]), s["embedded_rate_hz"]) for t, cs in cell["extra"]]
    ctx.generate_bursty(BurstConfig(electrodes=s["electrodes"], duration_s=s["duration_s"], seed=s["seed"],
                                    embedded=emb))
    types, times = ctx.download()
    assert len(types) == cell["n"]
    assert oracle.fnv_stream(types, times, cell["alphabet"]) == cell["stream_fnv"]
