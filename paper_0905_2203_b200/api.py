"""Python mirror of the reference's counting / mining API, backed by the
B200 kernels through the C-ABI (no CPU counting path exists).

Reference surface mirrored (paths relative to
/root/reference/proj/include/episodic):

  Event, IntervalConstraint, Episode, EventStream   types.hpp:20-134
  DataError, validate                               types.hpp:75-92
  count_fsm(stream, ep)                             fsm.hpp:101-106
  count_tracking(stream, index, ep, opt)            tracking.hpp:391-407
  count_mapconcat(stream, ep, segments, workers)    mapconcat.hpp:71-159
  generate_candidates(level, frequent, alpha, A)    miner.hpp:76-109
  MiningConfig / LevelResult / MiningResult / mine  miner.hpp:26-173
  write_mining_csv, format_episode                  miner.hpp:175-181, grammar.hpp:70-83
  GenConfig / Embedding / generate                  datagen.hpp:19-122

Errors map to the reference's exception types: std::invalid_argument ->
InvalidArgument (a ValueError), DataError -> DataError (a RuntimeError),
std::overflow_error -> OverflowError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Iterable, NamedTuple, Sequence

import numpy as np

from . import _native as N


class EpisodicError(RuntimeError):
    pass


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class DataError(RuntimeError):
    """episodic::DataError (E/types.hpp:75-80); `line` is the 1-based input
    line for event-file errors, 0 otherwise."""

    def __init__(self, msg: str, line: int = 0):
        super().__init__(msg)
        self.line = line


class Unsupported(EpisodicError):
    pass


def _raise(status: int, msg: str):
    if status == N.EPI_EINVAL:
        raise InvalidArgument(msg)
    if status == N.EPI_EDATA:
        line = 0
        if msg.startswith("line "):
            head = msg[5:].split(":", 1)[0]
            line = int(head) if head.isdigit() else 0
        raise DataError(msg, line)
    if status == N.EPI_EOVERFLOW:
        raise OverflowError(msg)
    if status == N.EPI_EUNSUPPORTED:
        raise Unsupported(msg)
    name = N.lib.epi_status_name(status).decode()
    raise EpisodicError(f"{name}: {msg}")


class Event(NamedTuple):
    type: int
    time: int


class IntervalConstraint(NamedTuple):
    """Half-open gap constraint: g admissible iff low < g <= high."""
    low: int
    high: int

    def contains_gap(self, gap: int) -> bool:
        return self.low < gap <= self.high


@dataclass(eq=True)
class Episode:
    types: list = field(default_factory=list)
    constraints: list = field(default_factory=list)

    def __post_init__(self):
        self.types = [int(t) for t in self.types]
        self.constraints = [IntervalConstraint(int(c[0]), int(c[1])) for c in self.constraints]

    def size(self) -> int:
        return len(self.types)

    def slice(self, first: int, length: int) -> "Episode":
        return Episode(self.types[first:first + length],
                       self.constraints[first:first + length - 1] if length > 1 else [])

    def key(self):
        return (tuple(self.types), tuple(self.constraints))


def validate(ep: Episode) -> None:
    """validate(Episode), E/types.hpp:82-92."""
    if not ep.types:
        raise InvalidArgument("episode must have at least one node")
    if len(ep.constraints) + 1 != len(ep.types):
        raise InvalidArgument("episode needs exactly N-1 constraints")
    for c in ep.constraints:
        if c.low < 0 or c.low >= c.high:
            raise InvalidArgument("interval constraint requires 0 <= low < high")


class EventStream:
    """Time-ordered SoA event stream (E/types.hpp:96-134). Validation of
    from_events happens on the device when the stream is loaded; it raises
    DataError with the reference's messages."""

    def __init__(self, types: np.ndarray, times: np.ndarray, alphabet: int):
        self.types_ = np.ascontiguousarray(types, dtype=np.uint32)
        self.times_ = np.ascontiguousarray(times, dtype=np.int64)
        if self.types_.shape != self.times_.shape:
            raise InvalidArgument("types and times must have the same length")
        self.alphabet_ = int(alphabet)

    @staticmethod
    def from_events(events: Iterable, alphabet_size: int) -> "EventStream":
        """EventStream::from_events (E/types.hpp:102-119): the first offending
        event decides the error, checks in the reference's order."""
        ev = list(events)
        types = np.array([int(e[0]) for e in ev], dtype=np.int64).reshape(-1)
        times = np.array([int(e[1]) for e in ev], dtype=np.int64).reshape(-1)
        bad_neg = times < 0
        bad_order = np.zeros_like(bad_neg)
        if len(ev) > 1:
            bad_order[1:] = times[1:] < times[:-1]
        bad_type = (types < 0) | (types >= alphabet_size)
        bad = bad_neg | bad_order | bad_type
        if bad.any():
            i = int(np.argmax(bad))
            if bad_neg[i]:
                raise DataError("negative event time")
            if bad_order[i]:
                raise DataError("event times must be non-decreasing")
            raise DataError("event type id out of range")
        return EventStream(types.astype(np.uint32), times, alphabet_size)

    @staticmethod
    def from_arrays(types, times, alphabet_size: int) -> "EventStream":
        return EventStream(types, times, alphabet_size)

    def size(self) -> int:
        return int(self.types_.shape[0])

    def __len__(self):
        return self.size()

    def empty(self) -> bool:
        return self.size() == 0

    def type_at(self, i: int) -> int:
        return int(self.types_[i])

    def time_at(self, i: int) -> int:
        return int(self.times_[i])

    def alphabet_size(self) -> int:
        return self.alphabet_

    def types(self) -> np.ndarray:
        return self.types_

    def times(self) -> np.ndarray:
        return self.times_


def episodes_to_csr(episodes: Sequence[Episode]) -> N.CSR:
    off = np.zeros(len(episodes) + 1, dtype=np.uint32)
    types, lo, hi = [], [], []
    for i, ep in enumerate(episodes):
        types.extend(ep.types)
        for c in ep.constraints:
            lo.append(c[0])
            hi.append(c[1])
        if len(ep.constraints) + 1 != len(ep.types) and ep.types:
            raise InvalidArgument("episode needs exactly N-1 constraints")
        off[i + 1] = off[i] + len(ep.types)
    return N.CSR(off, np.array(types, dtype=np.uint32), np.array(lo, dtype=np.int64),
                 np.array(hi, dtype=np.int64))


def csr_to_episodes(csr: N.CSR) -> list:
    return [Episode(*csr.episode(e)) for e in range(len(csr))]


class Context:
    """A device context (epi_ctx): a resident stream plus counting.
    Context(0) binds one device; Context(devices=[0, 1, ...]) one context
    over several devices of this process (epi_create_multi: stream
    replicated, candidates sharded, counts all-gathered per level by NCCL or
    device copies)."""

    def __init__(self, device: int = 0, devices=None):
        h = C.c_void_p()
        if devices is not None:
            devs = (C.c_int * len(devices))(*[int(d) for d in devices])
            st = N.lib.epi_create_multi(len(devices), devs, C.byref(h))
        else:
            st = N.lib.epi_create(device, C.byref(h))
        if st != N.EPI_OK:
            _raise(st, N.lib.epi_last_error(None).decode())
        self._h = h
        self._loaded = None
        self.device = device if devices is None else int(devices[0])
        self.world = int(N.lib.epi_world(h))
        self.uses_nccl = bool(N.lib.epi_uses_nccl(h))

    def close(self):
        if getattr(self, "_h", None):
            N.lib.epi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int):
        if st != N.EPI_OK:
            _raise(st, N.lib.epi_last_error(self._h).decode())

    def load(self, stream: EventStream):
        if self._loaded is stream:
            return
        self._loaded = None
        self._check(N.lib.epi_load_stream(self._h, N.ptr(stream.types_, C.c_uint32),
                                          N.ptr(stream.times_, C.c_int64), stream.size(),
                                          stream.alphabet_))
        self._loaded = stream

    def generate(self, cfg: "GenConfig"):
        """generate() (E/datagen.hpp:71-122) bit-exact on the device, loaded as
        this context's stream (epi_generate_stream)."""
        eps = [e.episode for e in cfg.embedded]
        csr = episodes_to_csr(eps) if eps else None
        rates = np.array([e.rate_hz for e in cfg.embedded], dtype=np.float64)
        self._loaded = None
        self._check(N.lib.epi_generate_stream(self._h, int(cfg.neurons), float(cfg.duration_s),
                                              float(cfg.base_rate_hz), int(cfg.seed) & ((1 << 64) - 1),
                                              C.byref(csr.struct) if csr is not None else None,
                                              N.ptr(rates, C.c_double) if len(rates) else None))

    def generate_bursty(self, cfg: "BurstConfig"):
        """The MEA-shaped bursty stream (generate_bursty_arrays) generated on
        the device and loaded as this context's stream
        (epi_generate_bursty_stream)."""
        eps = [e.episode for e in cfg.embedded]
        csr = episodes_to_csr(eps) if eps else None
        rates = np.array([e.rate_hz for e in cfg.embedded], dtype=np.float64)
        self._loaded = None
        self._check(N.lib.epi_generate_bursty_stream(
            self._h, int(cfg.electrodes), float(cfg.duration_s), float(cfg.base_rate_hz), float(cfg.rate_sigma),
            float(cfg.burst_rate_hz), float(cfg.burst_min_ms), float(cfg.burst_max_ms), float(cfg.burst_gain),
            int(cfg.seed) & ((1 << 64) - 1), C.byref(csr.struct) if csr is not None else None,
            N.ptr(rates, C.c_double) if len(rates) else None))

    def download(self):
        """(types, times) of the loaded stream (epi_stream_download)."""
        n = int(N.lib.epi_stream_size(self._h))
        types = np.zeros(n, dtype=np.uint32)
        times = np.zeros(n, dtype=np.int64)
        self._check(N.lib.epi_stream_download(self._h, N.ptr(types, C.c_uint32), N.ptr(times, C.c_int64)))
        return types, times

    @property
    def upload_bytes(self) -> int:
        """Host->device bytes of the last stream load (epi_stream_upload_bytes)."""
        return int(N.lib.epi_stream_upload_bytes(self._h))

    def load_arrays(self, types: np.ndarray, times: np.ndarray, alphabet: int):
        """Load from host arrays (pinned or pageable); returns nothing."""
        self._loaded = None
        self._check(N.lib.epi_load_stream(self._h, N.ptr(types, C.c_uint32), N.ptr(times, C.c_int64),
                                          int(types.shape[0]), alphabet))

    def load_file(self, path: str):
        """Load a binary event file (write_events_binary) straight from its
        mapping: no parse, pinned double-buffered H2D, from_events validation."""
        self._loaded = None
        self._check(N.lib.epi_load_stream_file(self._h, os.fsencode(path)))

    def load_device(self, d_types_ptr: int, d_times_ptr: int, n: int, alphabet: int):
        self._loaded = None
        self._check(N.lib.epi_load_stream_device(self._h, C.c_void_p(d_types_ptr),
                                                 C.c_void_p(d_times_ptr), n, alphabet))

    def count_csr(self, csr: N.CSR, threshold: int = 1, mode: int = N.MODE_EXACT,
                  with_frequent: bool = False, shard=None):
        """epi_count; shard = (rank, world, min_shard, allgather) runs
        epi_count_sharded (episode slices for >= min_shard episodes, time
        segments below; see shard.make_allgather)."""
        n = len(csr)
        counts = np.zeros(n, dtype=np.uint64)
        freq = np.zeros(n, dtype=np.uint8) if with_frequent else None
        stats = N.Stats()
        if shard is None:
            self._check(N.lib.epi_count(self._h, C.byref(csr.struct), int(threshold), int(mode),
                                        N.ptr(counts, C.c_uint64),
                                        N.ptr(freq, C.c_uint8) if freq is not None else None,
                                        C.byref(stats)))
        else:
            rank, world, min_shard, fn = shard

            def _cb(user, send, recv, nbytes, stream):
                try:
                    return int(fn(send, recv, int(nbytes), stream) or 0)
                except Exception as exc:  # noqa: BLE001 - reported as EPI_ENCCL
                    self.shard_error = exc
                    return 1
            cb = N.ALLGATHER_FN(_cb)
            sh = N.Shard(int(rank), int(world), int(min_shard), cb, None)
            self._check(N.lib.epi_count_sharded(self._h, C.byref(csr.struct), int(threshold), int(mode),
                                                C.byref(sh), N.ptr(counts, C.c_uint64),
                                                N.ptr(freq, C.c_uint8) if freq is not None else None,
                                                C.byref(stats)))
        self.last_stats = stats.as_dict()
        return (counts, freq) if with_frequent else counts

    def count(self, stream: EventStream, episodes: Sequence[Episode], threshold: int = 1,
              mode: int = N.MODE_EXACT):
        self.load(stream)
        return self.count_csr(episodes_to_csr(episodes), threshold, mode)

    def count_tracking_csr(self, csr: N.CSR, direction: int = 0):
        """Parallel local tracking + greedy on the device (epi_count_tracking)."""
        counts = np.zeros(len(csr), dtype=np.uint64)
        stats = N.Stats()
        self._check(N.lib.epi_count_tracking(self._h, C.byref(csr.struct), int(direction),
                                             N.ptr(counts, C.c_uint64), C.byref(stats)))
        self.last_stats = stats.as_dict()
        return counts

    def count_mapconcat_csr(self, csr: N.CSR, segments: int):
        """Exact counts with the caller's MapConcatenate segment count
        (epi_count_mapconcat); last_stats['segments'] is the count used."""
        counts = np.zeros(len(csr), dtype=np.uint64)
        stats = N.Stats()
        self._check(N.lib.epi_count_mapconcat(self._h, C.byref(csr.struct), int(segments),
                                              N.ptr(counts, C.c_uint64), C.byref(stats)))
        self.last_stats = stats.as_dict()
        return counts

    def find_occurrences_csr(self, csr: N.CSR, direction: int = 0):
        """(offsets, starts, ends) of every episode's occurrence intervals."""
        op, sp, ep = N.u64p(), N.i64p(), N.i64p()
        self._check(N.lib.epi_find_occurrences(self._h, C.byref(csr.struct), int(direction),
                                               C.byref(op), C.byref(sp), C.byref(ep)))
        try:
            n = len(csr)
            off = np.ctypeslib.as_array(op, shape=(n + 1,)).copy()
            tot = int(off[-1])
            s = np.ctypeslib.as_array(sp, shape=(max(tot, 1),))[:tot].copy()
            e = np.ctypeslib.as_array(ep, shape=(max(tot, 1),))[:tot].copy()
        finally:
            for ptr_ in (op, sp, ep):
                N.lib.epi_free(C.cast(ptr_, C.c_void_p))
        return off, s, e

    def mine_raw(self, threshold: int, bins: Sequence, max_level: int, mode: int = N.MODE_MINE,
                 shard=None):
        """Device-resident mine(). shard = (rank, world, min_shard, allgather)
        runs epi_mine_sharded: allgather(send_ptr, recv_ptr, bytes_per_rank,
        stream_ptr) -> 0 must all-gather the per-rank count slices (see
        shard.make_allgather)."""
        key = (tuple((int(b[0]), int(b[1])) for b in bins), int(threshold), int(max_level), int(mode))
        cached = getattr(self, "_mine_cfg", None)
        if cached is None or cached[0] != key:
            lo = np.array([b[0] for b in key[0]], dtype=np.int64)
            hi = np.array([b[1] for b in key[0]], dtype=np.int64)
            cfg_ = N.MineConfig(key[1], key[2], N.ptr(lo, C.c_int64), N.ptr(hi, C.c_int64), len(bins), key[3])
            self._mine_cfg = cached = (key, cfg_, lo, hi)  # arrays kept alive with the struct
        cfg = cached[1]
        res = N.MineResultOut()
        if shard is None:
            self._check(N.lib.epi_mine(self._h, C.byref(cfg), C.byref(res)))
        else:
            rank, world, min_shard, fn = shard

            def _cb(user, send, recv, nbytes, stream):
                try:
                    return int(fn(send, recv, int(nbytes), stream) or 0)
                except Exception as exc:  # noqa: BLE001 - reported as EPI_ENCCL
                    self.shard_error = exc
                    return 1
            cb = N.ALLGATHER_FN(_cb)  # kept alive for the duration of the call
            sh = N.Shard(int(rank), int(world), int(min_shard), cb, None)
            self._check(N.lib.epi_mine_sharded(self._h, C.byref(cfg), C.byref(sh), C.byref(res)))
        nl = int(res.n_levels)
        cands = (C.c_uint64 * nl).from_address(res.level_candidates)[:] if nl else []
        offs = (C.c_uint64 * (nl + 1)).from_address(res.level_offsets)[:] if res.level_offsets else [0]
        ms = (C.c_double * nl).from_address(res.level_ms)[:] if nl else []
        fr = res.frequent
        nf = int(fr.n_episodes)
        if nf:
            off = N.copy_addr(fr.offsets, nf + 1, np.uint32)
            nt = int(off[-1])
            csr = N.CSR(off, N.copy_addr(fr.types, nt, np.uint32), N.copy_addr(fr.low, nt - nf, np.int64),
                        N.copy_addr(fr.high, nt - nf, np.int64))
        else:
            csr = N.CSR(np.zeros(1, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.int64),
                        np.zeros(0, np.int64))
        counts = N.copy_addr(res.counts, nf, np.uint64)
        return cands, offs, ms, csr, counts, res.totals.as_dict()


_default = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def count_batch(stream: EventStream, episodes: Sequence[Episode]) -> np.ndarray:
    """Batch entry point (no reference equivalent: the reference loops over
    candidates, E/miner.hpp:145-154)."""
    for ep in episodes:
        validate(ep)
    return default_context().count(stream, episodes)


def count_fsm(stream: EventStream, ep: Episode) -> int:
    """count_fsm, E/fsm.hpp:101-106."""
    validate(ep)
    return int(default_context().count(stream, [ep])[0])


@dataclass
class TrackingStats:
    """TrackingStats, E/tracking.hpp:41-45 (flag_retries stays 0: the device
    compacts with a block scan, no slabs)."""
    sort_fallbacks: int = 0
    flag_retries: int = 0
    items_tracked: int = 0


@dataclass
class MapConcatStats:
    """MapConcatStats, E/mapconcat.hpp:26-30: the device's FRESH segment
    machines (precomputed), those the concat walk used as they were (hits)
    and the boundary machines it re-ran (patches)."""
    machines_precomputed: int = 0
    machine_hits: int = 0
    patches: int = 0


@dataclass
class TrackingOptions:
    """TrackingOptions, E/tracking.hpp:33-39. direction is used; the CPU
    compaction strategy, workers and slab width have no device meaning (the
    device compacts with a block scan) and are accepted for parity."""
    direction: str = "forward"
    strategy: str = "count_scan_write"
    workers: int = 1
    flag_slots: int = 32


def _direction(opt) -> int:
    d = getattr(opt, "direction", "forward") if opt is not None else "forward"
    return 1 if str(d).lower().endswith("backward") else 0


def count_tracking(stream: EventStream, index, ep: Episode, opt=None, stats=None) -> int:
    """count_tracking, E/tracking.hpp:391-407, on the device: parallel local
    tracking + greedy_schedule (equal to count_fsm on every input). `index`
    is accepted for signature parity (the device builds its own)."""
    validate(ep)
    ctx = default_context()
    ctx.load(stream)
    c = int(ctx.count_tracking_csr(episodes_to_csr([ep]), _direction(opt))[0])
    if stats is not None:
        stats.items_tracked += int(ctx.last_stats["items_tracked"])
        stats.sort_fallbacks += int(ctx.last_stats["sort_fallbacks"])
    return c


def find_occurrences(stream: EventStream, index, ep: Episode, opt=None, stats=None) -> list:
    """find_occurrences, E/tracking.hpp:330-367, on the device: the
    representative occurrence intervals [(start, end)] in the reference's
    order."""
    validate(ep)
    ctx = default_context()
    ctx.load(stream)
    off, s, e = ctx.find_occurrences_csr(episodes_to_csr([ep]), _direction(opt))
    return [(int(a), int(b)) for a, b in zip(s, e)]


def count_mapconcat(stream: EventStream, ep: Episode, segments: int, workers: int = 1,
                    stats=None) -> int:
    """count_mapconcat, E/mapconcat.hpp:71-159: the device MapConcatenate
    counter with `segments` time segments (epi_count_mapconcat; clamped to
    what the stream allows). `workers` has no device meaning."""
    validate(ep)
    if segments < 1:
        raise InvalidArgument("count_mapconcat: segments must be >= 1")
    if stream.size() == 0:
        return 0
    ctx = default_context()
    ctx.load(stream)
    c = int(ctx.count_mapconcat_csr(episodes_to_csr([ep]), segments)[0])
    if stats is not None:
        P = max(int(ctx.last_stats["segments"]), 1)
        stats.machines_precomputed = P
        stats.patches = int(ctx.last_stats["patches"])
        stats.machine_hits = P - min(P, stats.patches)
    return c


def generate_candidates(level: int, frequent: Sequence[Episode], alphabet: Sequence,
                        alphabet_size: int) -> list:
    """generate_candidates, E/miner.hpp:76-109 (host C++ join)."""
    csr = episodes_to_csr(list(frequent)) if frequent else N.CSR(np.zeros(1, np.uint32), [], [], [])
    lo = np.array([c[0] for c in alphabet], dtype=np.int64)
    hi = np.array([c[1] for c in alphabet], dtype=np.int64)
    out = N.EpisodeBatch()
    st = N.lib.epi_generate_candidates(None, int(level), C.byref(csr.struct), N.ptr(lo, C.c_int64),
                                       N.ptr(hi, C.c_int64), len(lo), int(alphabet_size), C.byref(out))
    if st != N.EPI_OK:
        _raise(st, N.lib.epi_last_error(None).decode())
    return csr_to_episodes(N.CSR.from_struct(out))


@dataclass
class MiningConfig:
    """MiningConfig, E/miner.hpp:26-37. `backend`, `strategy_switch_level`,
    `tracking`, `segments` and `workers` are accepted for parity; the device
    counter replaces all of them. `mode` selects two-pass elimination."""
    threshold: int = 1
    constraint_alphabet: list = field(default_factory=list)
    max_level: int = 16
    strategy_switch_level: int = 3
    backend: str = "device"
    tracking: object = None
    segments: int = 4
    workers: int = 1
    mode: int = N.MODE_MINE


@dataclass
class LevelResult:
    level: int = 0
    candidates: int = 0
    frequent: list = field(default_factory=list)
    elapsed_ms: float = 0.0


@dataclass
class MiningResult:
    levels: list = field(default_factory=list)
    stats: dict = field(default_factory=dict)


def mine(stream: EventStream, cfg: MiningConfig, ctx: Context | None = None) -> MiningResult:
    """mine, E/miner.hpp:114-173, one device count per level."""
    ctx = ctx or default_context()
    ctx.load(stream)
    cands, offs, ms, csr, counts, totals = ctx.mine_raw(cfg.threshold, cfg.constraint_alphabet,
                                                        cfg.max_level, cfg.mode)
    eps = csr_to_episodes(csr)
    levels = []
    for i in range(len(cands)):
        fr = [(eps[j], int(counts[j])) for j in range(offs[i], offs[i + 1])]
        levels.append(LevelResult(i + 1, cands[i], fr, ms[i]))
    return MiningResult(levels, totals)


def format_episode(ep: Episode, names=None) -> str:
    """format_episode, E/grammar.hpp:70-83 (numeric symbol table by default)."""
    out = []
    for i, t in enumerate(ep.types):
        if i:
            c = ep.constraints[i - 1]
            out.append(f"-({c.low},{c.high}]-")
        out.append(str(t) if names is None else names[t])
    return "".join(out)


def write_mining_csv(result: MiningResult, names=None) -> str:
    """write_mining_csv, E/miner.hpp:175-181."""
    lines = ["level,episode,count"]
    for lvl in result.levels:
        for ep, cnt in lvl.frequent:
            lines.append(f"{lvl.level},{format_episode(ep, names)},{cnt}")
    return "\n".join(lines) + "\n"


@dataclass
class Embedding:
    episode: Episode
    rate_hz: float = 1.0


@dataclass
class GenConfig:
    """GenConfig, E/datagen.hpp:19-25."""
    neurons: int = 64
    duration_s: float = 100.0
    base_rate_hz: float = 20.0
    embedded: list = field(default_factory=list)
    seed: int = 0


def generate_arrays(cfg: GenConfig):
    """generate(), E/datagen.hpp:71-122, as (types u32, times i64) arrays."""
    eps = [e.episode for e in cfg.embedded]
    csr = episodes_to_csr(eps) if eps else None
    rates = np.array([e.rate_hz for e in cfg.embedded], dtype=np.float64)
    tp, tm, n = N.u32p(), N.i64p(), C.c_uint64()
    st = N.lib.epi_generate(int(cfg.neurons), float(cfg.duration_s), float(cfg.base_rate_hz),
                            int(cfg.seed) & ((1 << 64) - 1),
                            C.byref(csr.struct) if csr is not None else None,
                            N.ptr(rates, C.c_double) if len(rates) else None,
                            C.byref(tp), C.byref(tm), C.byref(n))
    return _take_stream(st, tp, tm, n)


def _take_stream(st, tp, tm, n):
    if st != N.EPI_OK:
        _raise(st, N.lib.epi_last_error(None).decode())
    try:
        cnt = int(n.value)
        types = np.ctypeslib.as_array(tp, shape=(max(cnt, 1),))[:cnt].copy()
        times = np.ctypeslib.as_array(tm, shape=(max(cnt, 1),))[:cnt].copy()
    finally:
        N.lib.epi_free(C.cast(tp, C.c_void_p))
        N.lib.epi_free(C.cast(tm, C.c_void_p))
    return types, times


@dataclass
class BurstConfig:
    """MEA-shaped bursty stream (no reference
    counterpart): lognormal per-electrode rates, network bursts, embedded
    episodes."""
    electrodes: int = 60
    duration_s: float = 100.0
    base_rate_hz: float = 5.0
    rate_sigma: float = 0.5
    burst_rate_hz: float = 0.2
    burst_min_ms: float = 100.0
    burst_max_ms: float = 300.0
    burst_gain: float = 20.0
    embedded: list = field(default_factory=list)
    seed: int = 0


def generate_bursty_arrays(cfg: BurstConfig):
    eps = [e.episode for e in cfg.embedded]
    csr = episodes_to_csr(eps) if eps else None
    rates = np.array([e.rate_hz for e in cfg.embedded], dtype=np.float64)
    tp, tm, n = N.u32p(), N.i64p(), C.c_uint64()
    st = N.lib.epi_generate_bursty(int(cfg.electrodes), float(cfg.duration_s), float(cfg.base_rate_hz),
                                   float(cfg.rate_sigma), float(cfg.burst_rate_hz),
                                   float(cfg.burst_min_ms), float(cfg.burst_max_ms),
                                   float(cfg.burst_gain), int(cfg.seed) & ((1 << 64) - 1),
                                   C.byref(csr.struct) if csr is not None else None,
                                   N.ptr(rates, C.c_double) if len(rates) else None,
                                   C.byref(tp), C.byref(tm), C.byref(n))
    return _take_stream(st, tp, tm, n)


def random_episodes_csr(seed: int, count: int, nodes: int, alphabet: int, bins) -> N.CSR:
    """Seeded synthetic candidates (epi_random_episodes: one mt19937_64
    stream, per episode `nodes` types % alphabet then nodes-1 indices into
    `bins`), as a CSR batch."""
    types = np.zeros(count * nodes, dtype=np.uint32)
    bidx = np.zeros(max(count * (nodes - 1), 1), dtype=np.uint32)
    st = N.lib.epi_random_episodes(int(seed) & ((1 << 64) - 1), int(count), int(nodes), int(alphabet),
                                   len(bins), N.ptr(types, C.c_uint32), N.ptr(bidx, C.c_uint32))
    if st != 0:
        _raise(st, N.lib.epi_last_error(None).decode())
    bidx = bidx[:count * (nodes - 1)]
    lo = np.array([b[0] for b in bins], np.int64)[bidx]
    hi = np.array([b[1] for b in bins], np.int64)[bidx]
    off = (np.arange(count + 1, dtype=np.uint64) * nodes).astype(np.uint32)
    return N.CSR(off, types, lo, hi)


def generate(cfg: GenConfig) -> EventStream:
    types, times = generate_arrays(cfg)
    return EventStream(types, times, cfg.neurons)


class LoadedStream(NamedTuple):
    """LoadedStream, E/io.hpp:14-17: the stream plus its symbol names (id
    order, first-seen)."""
    stream: EventStream
    symbols: list


def load_stream(text) -> LoadedStream:
    """load_stream, E/io.hpp:22-56, parsed natively (multi-threaded C++ in
    csrc/io.cpp): `<name>,<int_ms>` per line; '#' comments, blank lines and
    CRLF tolerated; DataError with the reference's message and `.line`."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    tp, tm, n = N.u32p(), N.i64p(), C.c_uint64()
    names_p, alpha = C.c_void_p(), C.c_uint32()
    st = N.lib.epi_parse_events(data, len(data), C.byref(tp), C.byref(tm), C.byref(n),
                                C.byref(names_p), C.byref(alpha))
    if st != N.EPI_OK:
        _raise(st, N.lib.epi_last_error(None).decode())
    try:
        joined = C.string_at(names_p.value).decode() if names_p.value else ""
    finally:
        N.lib.epi_free(names_p)
    types, times = _take_stream(st, tp, tm, n)
    names = joined.split("\n") if alpha.value else []
    return LoadedStream(EventStream(types, times, int(alpha.value)), names)


def load_stream_file(path: str) -> LoadedStream:
    """load_stream_file, E/io.hpp:58-62."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise DataError(f"cannot open event file '{path}'") from None
    return load_stream(data)


def serialize_stream(stream: EventStream, symbols=None) -> str:
    """serialize_stream, E/io.hpp:64-67 (numeric names by default, like
    SymbolTable::numeric)."""
    types, times = stream.types(), stream.times()
    if symbols is None:
        names = types.astype(str)
    else:
        names = np.asarray(list(symbols), dtype=object)[types]
    if len(types) == 0:
        return ""
    return "\n".join(f"{a},{b}" for a, b in zip(names.tolist(), times.tolist())) + "\n"


def write_events_binary(path: str, types: np.ndarray, times: np.ndarray, alphabet: int) -> None:
    """Binary event file (EPIEVT01, include/episodic_b200.h; no reference
    counterpart): the SoA epi_load_stream takes."""
    types = np.ascontiguousarray(types, dtype=np.uint32)
    times = np.ascontiguousarray(times, dtype=np.int64)
    if types.shape != times.shape:
        raise InvalidArgument("types and times differ in length")
    st = N.lib.epi_write_events(os.fsencode(path), N.ptr(types, C.c_uint32), N.ptr(times, C.c_int64),
                                int(types.shape[0]), int(alphabet))
    if st != N.EPI_OK:
        _raise(st, N.lib.epi_last_error(None).decode())


def read_events_binary(path: str):
    """(types, times, alphabet) of a binary event file; DataError on a
    missing, foreign or truncated file."""
    tp, tm, n, alpha = N.u32p(), N.i64p(), C.c_uint64(), C.c_uint32()
    st = N.lib.epi_read_events(os.fsencode(path), C.byref(tp), C.byref(tm), C.byref(n), C.byref(alpha))
    types, times = _take_stream(st, tp, tm, n)
    return types, times, int(alpha.value)
