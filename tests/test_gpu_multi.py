"""epi_create_multi: one context over several devices of the process (one
engine and stream per device, candidates sharded, counts all-gathered per
level). The GPU box has one device, so groups repeat device 0 - the
device-copy exchange - and a one-device group runs NCCL's path setup; every
result must equal the single-device context's (and the reference's CSV for
mining)."""
import numpy as np
import pytest

from helpers import csr_of
from paper_0905_2203_b200 import (MODE_EXACT, MODE_MINE, Context, EventStream, GenConfig, MiningConfig,
                                  generate_arrays, mine, write_mining_csv)

pytestmark = pytest.mark.gpu

BINS = [(0, 5), (5, 10), (10, 15)]


def _cands(rng, n, a=64):
    return [([int(x) for x in rng.integers(0, a, 3)], [BINS[int(b)] for b in rng.integers(0, 3, 2)])
            for _ in range(n)]


@pytest.mark.parametrize("world", [1, 2, 3])
def test_multi_count_equals_single(ctx, world):
    types, times = generate_arrays(GenConfig(64, 2_000_000 / (64 * 20), 20, [], 61))
    rng = np.random.default_rng(world)
    many = csr_of(_cands(rng, 30000))  # episode-sharded (>= 4096 per rank)
    few = csr_of(_cands(rng, 50))      # time-sharded (segments per rank)
    ctx.load_arrays(types, times, 64)
    want_many, want_few = ctx.count_csr(many), ctx.count_csr(few)
    want_mine = ctx.count_csr(many, threshold=30, mode=MODE_MINE)
    m = Context(devices=[0] * world)
    try:
        assert m.world == world
        m.load_arrays(types, times, 64)
        np.testing.assert_array_equal(m.count_csr(many), want_many)
        np.testing.assert_array_equal(m.count_csr(few), want_few)
        np.testing.assert_array_equal(m.count_csr(many, threshold=30, mode=MODE_MINE), want_mine)
    finally:
        m.close()


@pytest.mark.parametrize("world", [2, 3])
def test_multi_mine_equals_reference(golden_configs, world):
    """cfg2 mining through a multi-device context: level 3 (142,228
    candidates) is sharded; the CSV equals the reference's mine()."""
    from bench import make_stream
    types, times, a = make_stream("cfg2")
    g = golden_configs["cfg2"]
    m = Context(devices=[0] * world)
    try:
        cfg = MiningConfig(threshold=250, constraint_alphabet=BINS, max_level=4, mode=MODE_MINE)
        r = mine(EventStream(types, times, a), cfg, ctx=m)
        assert write_mining_csv(r) == g["csv"]
        assert [lv.candidates for lv in r.levels] == g["level_candidates"]
    finally:
        m.close()


def test_multi_errors_are_reported(ctx):
    m = Context(devices=[0, 0])
    try:
        m.load_arrays(np.array([0, 1], np.uint32), np.array([5, 3], np.int64), 2)
    except Exception as e:  # noqa: BLE001
        assert "non-decreasing" in str(e)
    else:
        raise AssertionError("bad stream accepted")
    finally:
        m.close()
