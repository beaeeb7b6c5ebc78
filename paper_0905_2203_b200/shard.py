"""Episode-sharded counting and mining across GPUs (one process per GPU).

Candidates of a level are independent units: rank r of G takes
the contiguous slice [r*n/G, (r+1)*n/G) of the level's candidate list,
counts it on its own device, and one all_gather of the u64 counts (padded to
equal slices) gives every rank the full level result in candidate order. The
host then thresholds and joins the next level identically on every rank, so
the frequent sets stay bit-identical across ranks without further exchange.
The stream is replicated (each rank loads it into its own HBM).

The counting function is injected: the product passes the device counter
(Context.count_csr); the CPU tests pass the oracle with the gloo backend.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Sequence

import numpy as np

from ._native import CSR, MODE_EXACT


def shard_bounds(n: int, world: int, rank: int) -> tuple:
    return (n * rank // world, n * (rank + 1) // world)


def slice_csr(csr: CSR, lo: int, hi: int) -> CSR:
    off = csr.offsets
    b, e = int(off[lo]), int(off[hi])
    cb, ce = b - lo, e - hi
    return CSR(off[lo:hi + 1] - off[lo], csr.types[b:e], csr.low[cb:ce], csr.high[cb:ce])


def allgather_counts(local: np.ndarray, n: int, group=None, device=None) -> np.ndarray:
    """all_gather of per-rank u64 count slices (padded to the largest slice)
    -> the full count vector in candidate order on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    width = max(hi - lo for lo, hi in (shard_bounds(n, world, r) for r in range(world)))
    buf = torch.zeros(width, dtype=torch.int64, device=device)
    if len(local):
        buf[:len(local)] = torch.from_numpy(local.astype(np.uint64).view(np.int64)).to(buf.device)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = np.empty(n, dtype=np.uint64)
    for r, part in enumerate(parts):
        lo, hi = shard_bounds(n, world, r)
        out[lo:hi] = part[:hi - lo].cpu().numpy().view(np.uint64)
    return out


def count_sharded(csr: CSR, count_fn: Callable, group=None, device=None, threshold: int = 1,
                  mode: int = MODE_EXACT) -> np.ndarray:
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    n = len(csr)
    lo, hi = shard_bounds(n, world, rank)
    local = count_fn(slice_csr(csr, lo, hi), threshold, mode) if hi > lo else np.zeros(0, np.uint64)
    return allgather_counts(np.asarray(local, dtype=np.uint64), n, group, device)


class _RawDevice:
    """A device byte range as a __cuda_array_interface__ object (zero-copy
    torch view of an engine buffer)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def make_allgather(group=None, memory: str = "cuda", device=None):
    """The all-gather callback of epi_mine_sharded (Context.mine_raw(shard=...)).

    memory="cuda":   the pointers are device buffers on the engine's stream;
                     NCCL all_gather_into_tensor enqueued on that stream
                     (torch.cuda.ExternalStream), no host round trip.
    memory="staged": device buffers, gathered through host copies (gloo;
                     functional runs of several ranks on one GPU).
    memory="host":   the pointers are host memory (CPU tests of the plumbing).
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)

    def host_view(ptr, nbytes):
        return torch.from_numpy(np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(int(ptr))))

    def fn(send, recv, nbytes, stream):
        if memory == "host":
            src = host_view(send, nbytes)
            parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, src.clone(), group=group)
            host_view(recv, nbytes * world).copy_(torch.cat(parts))
            return 0
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        s = torch.cuda.ExternalStream(int(stream), device=dev)
        with torch.cuda.stream(s):
            src = torch.as_tensor(_RawDevice(send, nbytes), device=dev)
            dst = torch.as_tensor(_RawDevice(recv, nbytes * world), device=dev)
            if memory == "cuda":
                dist.all_gather_into_tensor(dst, src, group=group)
            else:
                h = src.cpu()
                parts = [torch.empty_like(h) for _ in range(world)]
                dist.all_gather(parts, h, group=group)
                dst.copy_(torch.cat(parts))
                s.synchronize()
        return 0
    return fn


def mine_sharded(alphabet_size: int, threshold: int, bins: Sequence, max_level: int,
                 count_fn: Callable, group=None, device=None, mode: int = MODE_EXACT):
    """mine() (E/miner.hpp:114-173) with each level's counting block
    episode-sharded across the ranks of `group`. Returns
    [(level, n_candidates, [(types, constraints, count), ...]), ...]."""
    from .api import Episode, episodes_to_csr, generate_candidates
    from ._native import COUNT_PRUNED
    levels = []
    frequent: list = []
    for level in range(1, max_level + 1):
        cands = generate_candidates(level, frequent, bins, alphabet_size)
        if not cands:
            break
        csr = episodes_to_csr(cands)
        counts = count_sharded(csr, count_fn, group, device, threshold,
                               MODE_EXACT if level == 1 else mode)
        keep = [(c, int(k)) for c, k in zip(cands, counts)
                if int(k) != COUNT_PRUNED and int(k) >= threshold]
        levels.append((level, len(cands), [(c.types, c.constraints, k) for c, k in keep]))
        frequent = [Episode(c.types, c.constraints) for c, _ in keep]
        if not frequent:
            break
    return levels
