"""Multi-rank path on CPU: world_size 2 over gloo. Each rank counts its
episode shard (the oracle port stands in for the device counter, which
needs a GPU) and the per-level all_gather reassembles the counts; the
sharded mining result must equal the reference's single-process mine()."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cfg2_stream():
    from paper_0905_2203_b200 import Embedding, Episode, GenConfig, generate_arrays
    b = [(0, 5), (5, 10), (10, 15)]
    eps = [([0, 1, 2, 3], [b[1]] * 3), ([4, 5, 6, 7], [b[0], b[1], b[2]]),
           ([8, 9, 10, 11], [b[2], b[0], b[1]]), ([12, 13, 14, 15], [b[1], b[2], b[0]])]
    return generate_arrays(GenConfig(26, 60, 32, [Embedding(Episode(t, c), 5.0) for t, c in eps], 1))


def _worker(rank, world, port, queue, task):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_0905_2203_b200.shard import count_sharded, mine_sharded, shard_bounds
        if task == "allgather":
            # the epi_mine_sharded callback contract on host memory: send = this
            # rank's s u64, recv = world * s u64 in rank order
            from paper_0905_2203_b200.shard import make_allgather
            s = 37
            send = (np.arange(s, dtype=np.uint64) + 1000 * rank).astype(np.uint64)
            recv = np.zeros(s * world, dtype=np.uint64)
            fn = make_allgather(memory="host")
            rc = fn(send.ctypes.data, recv.ctypes.data, s * 8, 0)
            want = np.concatenate([np.arange(s, dtype=np.uint64) + 1000 * r for r in range(world)])
            queue.put((rank, rc == 0 and bool(np.array_equal(recv, want)), True))
        elif task == "count":
            rng = np.random.default_rng(3)
            times = np.cumsum(rng.integers(0, 5, 4000)).astype(np.int64)
            types = rng.integers(0, 6, 4000).astype(np.uint32)
            from helpers import csr_of
            eps = [([int(x) for x in rng.integers(0, 6, 3)], [(0, 5), (2, 7)]) for _ in range(37)]
            csr = csr_of(eps)
            seen = []

            def count_fn(part, threshold, mode):
                seen.append(len(part))
                return oracle.count_batch(types, times, part.offsets, part.types, part.low, part.high)
            got = count_sharded(csr, count_fn)
            want = oracle.count_batch(types, times, csr.offsets, csr.types, csr.low, csr.high)
            lo, hi = shard_bounds(37, world, rank)
            queue.put((rank, bool(np.array_equal(got, want)), seen == [hi - lo]))
        else:
            types, times = _cfg2_stream()

            def count_fn(part, threshold, mode):
                return oracle.count_batch(types, times, part.offsets, part.types, part.low, part.high,
                                          threads=2)
            levels = mine_sharded(26, 250, [(0, 5), (5, 10), (10, 15)], 3, count_fn)
            lines = ["level,episode,count"]
            for lv, _, fr in levels:
                for t, c, k in fr:
                    s = str(t[0]) + "".join(f"-({lo},{hi}]-{x}" for (lo, hi), x in zip(c, t[1:]))
                    lines.append(f"{lv},{s},{k}")
            queue.put((rank, "\n".join(lines) + "\n", [n for _, n, _ in levels]))
    finally:
        dist.destroy_process_group()


def _run(task, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, task)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


def test_allgather_callback_world2():
    for rank, ok, _ in _run("allgather"):
        assert ok, rank


def test_sharded_count_world2():
    for rank, equal, sliced in _run("count"):
        assert equal and sliced, rank


@pytest.mark.timeout(900)
def test_sharded_mining_world2_matches_reference():
    g = load_golden("configs.json")["cfg2"]
    want_lines = [l for l in g["csv"].splitlines() if not l.startswith("4,")]
    results = _run("mine")
    for rank, csv, cands in results:
        assert cands == g["level_candidates"][:3], rank
        assert csv.splitlines() == want_lines, rank
