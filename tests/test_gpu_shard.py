"""epi_mine_sharded on one GPU: two contexts (ranks) in two threads, the
all-gather callback exchanging device slices through a barrier. Every
rank's result must equal the unsharded device miner's and the reference's
cfg2 CSV; the callback must see the C-ABI's slice contract (s * 8 bytes per
rank, recv = world * s u64)."""
import threading

import numpy as np
import pytest

from paper_0905_2203_b200 import MODE_EXACT, MODE_MINE, Context
from paper_0905_2203_b200.shard import _RawDevice

pytestmark = pytest.mark.gpu

BINS = [(0, 5), (5, 10), (10, 15)]


def _cfg2():
    from paper_0905_2203_b200 import Embedding, Episode, GenConfig, generate_arrays
    b = BINS
    eps = [([0, 1, 2, 3], [b[1]] * 3), ([4, 5, 6, 7], [b[0], b[1], b[2]]),
           ([8, 9, 10, 11], [b[2], b[0], b[1]]), ([12, 13, 14, 15], [b[1], b[2], b[0]])]
    return generate_arrays(GenConfig(26, 60, 32, [Embedding(Episode(t, c), 5.0) for t, c in eps], 1))


def _threaded_mine(types, times, world, min_shard, mode, max_level=4, threshold=250):
    import torch
    ctxs = [Context(0) for _ in range(world)]
    for c in ctxs:
        c.load_arrays(types, times, 26)
    barrier = threading.Barrier(world)
    slices, calls, out, errs = {}, [], [None] * world, []

    def make_fn(r):
        def fn(send, recv, nbytes, stream):
            torch.cuda.ExternalStream(int(stream)).synchronize()
            slices[r] = torch.as_tensor(_RawDevice(send, nbytes), device="cuda").clone()
            calls.append((r, nbytes))
            barrier.wait()
            dst = torch.as_tensor(_RawDevice(recv, nbytes * world), device="cuda")
            dst.copy_(torch.cat([slices[q] for q in range(world)]))
            torch.cuda.synchronize()
            barrier.wait()
            return 0
        return fn

    def run(r):
        try:
            out[r] = ctxs[r].mine_raw(threshold, BINS, max_level, mode, shard=(r, world, min_shard, make_fn(r)))
        except Exception as exc:  # surfaced below
            errs.append(exc)
            barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    for c in ctxs:
        c.close()
    assert not errs, errs
    return out, calls


def _csv(res):
    cands, offs, ms, csr, counts, st = res
    lines = []
    for lv in range(len(cands)):
        for i in range(offs[lv], offs[lv + 1]):
            t, c = csr.episode(i)
            lines.append((lv + 1, tuple(t), tuple(c), int(counts[i])))
    return cands, lines


@pytest.mark.parametrize("world,mode", [(2, MODE_MINE), (3, MODE_MINE), (2, MODE_EXACT)])
def test_sharded_mining_equals_unsharded(ctx, world, mode):
    types, times = _cfg2()
    ctx.load_arrays(types, times, 26)
    want = _csv(ctx.mine_raw(250, BINS, 4, mode))
    got, calls = _threaded_mine(types, times, world, 64, mode)
    for r in range(world):
        assert _csv(got[r]) == want, r
    # levels 2..4 (2,028 / 142,228 / 4 candidates): 4 < min(64, world^2) is
    # not sharded; the others are, one callback per rank each, s*8 bytes
    sizes = sorted({nb for _, nb in calls})
    assert sizes == sorted({(n + world - 1) // world * 8 for n in (2028, 142228)})
    assert len(calls) == 2 * world


def test_sharded_mining_matches_reference_csv(golden_configs):
    g = golden_configs["cfg2"]
    types, times = _cfg2()
    got, _ = _threaded_mine(types, times, 2, 64, MODE_MINE)
    for r in range(2):
        cands, lines = _csv(got[r])
        assert cands == g["level_candidates"]
        csv = ["level,episode,count"] + [
            f"{lv}," + str(t[0]) + "".join(f"-({lo},{hi}]-{x}" for (lo, hi), x in zip(c, t[1:])) + f",{k}"
            for lv, t, c, k in lines]
        assert csv == g["csv"].splitlines()


def test_sharded_callback_failure_is_enccl():
    from paper_0905_2203_b200 import EpisodicError
    types, times = _cfg2()
    c = Context(0)
    c.load_arrays(types, times, 26)
    with pytest.raises(EpisodicError, match="all-gather"):
        c.mine_raw(250, BINS, 3, MODE_MINE, shard=(0, 2, 16, lambda *a: 1))
    c.close()


def test_allgather_callback_nccl_plumbing():
    """make_allgather(memory="cuda") on hardware: device pointers wrapped as
    torch tensors (__cuda_array_interface__), NCCL all_gather_into_tensor
    enqueued on the engine's stream (ExternalStream). World 1 (one GPU per
    gpurun box): recv must equal send, ordered on that stream."""
    import socket

    import torch
    import torch.distributed as dist
    from paper_0905_2203_b200.shard import make_allgather
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        fn = make_allgather(memory="cuda", device=torch.device("cuda", 0))
        st = torch.cuda.Stream()
        send = torch.arange(1000, dtype=torch.int64, device="cuda") * 7
        recv = torch.zeros(1000, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        assert fn(send.data_ptr(), recv.data_ptr(), 8000, st.cuda_stream) == 0
        st.synchronize()
        assert torch.equal(send, recv)
    finally:
        dist.destroy_process_group()


def _threaded(world, fn_per_rank):
    """Run fn_per_rank(rank, allgather_fn) in `world` threads with a barrier
    all-gather over device pointers; returns the per-rank results."""
    import torch
    barrier = threading.Barrier(world)
    slices, out, errs = {}, [None] * world, []

    def make_fn(r):
        def fn(send, recv, nbytes, stream):
            torch.cuda.ExternalStream(int(stream)).synchronize()
            slices[r] = torch.as_tensor(_RawDevice(send, nbytes), device="cuda").clone()
            barrier.wait()
            dst = torch.as_tensor(_RawDevice(recv, nbytes * world), device="cuda")
            dst.copy_(torch.cat([slices[q] for q in range(world)]))
            torch.cuda.synchronize()
            barrier.wait()
            return 0
        return fn

    def run(r):
        try:
            out[r] = fn_per_rank(r, make_fn(r))
        except Exception as exc:
            errs.append(exc)
            barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    return out


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", ["time", "time_mine", "time_forced", "episode"])
def test_sharded_count_equals_unsharded(ctx, world, case, monkeypatch):
    """epi_count_sharded: few episodes over a long stream shard the
    MapConcatenate segments by time (records all-gathered, walked on every
    rank); many episodes shard by episode. Every rank's counts == the
    unsharded device counts (and the oracle port on a subset)."""
    import oracle
    from helpers import csr_of
    from paper_0905_2203_b200 import GenConfig, generate_arrays
    types, times = generate_arrays(GenConfig(64, 1_000_000 / (64 * 20), 20, [], 51))
    rng = np.random.default_rng(world)
    nep = 2000 if case == "episode" else 40
    eps = [([int(x) for x in rng.integers(0, 64, 3)], [BINS[int(b)] for b in rng.integers(0, 3, 2)])
           for _ in range(nep)]
    csr = csr_of(eps)
    mode = MODE_MINE if case == "time_mine" else MODE_EXACT
    thr = 40 if case == "time_mine" else 1
    if case == "time_forced":
        monkeypatch.setenv("EPI_FORCE_SEGMENTS", "7")
    ctx.load_arrays(types, times, 64)
    want = ctx.count_csr(csr, thr, mode)

    def per_rank(r, fn):
        c = Context(0)
        c.load_arrays(types, times, 64)
        got = c.count_csr(csr, thr, mode, shard=(r, world, 1000, fn))
        st = c.last_stats
        c.close()
        return got, st
    res = _threaded(world, per_rank)
    for r, (got, st) in enumerate(res):
        np.testing.assert_array_equal(got, want, err_msg=f"rank {r}")
        if case.startswith("time"):
            assert st["segments"] >= world
    sub = csr_of(eps[:8])
    exact = oracle.count_batch(types, times, sub.offsets, sub.types, sub.low, sub.high, threads=8)
    if mode == MODE_EXACT:
        np.testing.assert_array_equal(res[0][0][:8], exact)
