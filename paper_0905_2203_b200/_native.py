"""ctypes binding of the C-ABI in include/episodic_b200.h.

The shared library is built in-tree (paper_0905_2203_b200/_lib/) by
`__graft_entry__.build()`. There is no fallback: if the library is missing
the import fails loudly, so nothing can silently count on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# EPI_LIB: an alternative in-tree build of the library (kernel experiments)
LIB_PATH = os.environ.get("EPI_LIB") or os.path.join(_HERE, "_lib", "libepisodic_b200.so")

EPI_OK, EPI_EINVAL, EPI_EDATA, EPI_EOVERFLOW, EPI_ECUDA, EPI_ENCCL, EPI_ENOMEM, EPI_EUNSUPPORTED = range(8)
MODE_EXACT, MODE_MINE = 0, 1
COUNT_PRUNED = (1 << 64) - 1

u32p = C.POINTER(C.c_uint32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
u8p = C.POINTER(C.c_uint8)
f64p = C.POINTER(C.c_double)


class EpisodeBatch(C.Structure):
    _fields_ = [("n_episodes", C.c_uint64), ("offsets", u32p), ("types", u32p),
                ("low", i64p), ("high", i64p)]


class Stats(C.Structure):
    _fields_ = [("episodes", C.c_uint64), ("pass1_groups", C.c_uint64),
                ("pass2_episodes", C.c_uint64), ("pruned", C.c_uint64),
                ("segments", C.c_uint64), ("patches", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("map_launches", C.c_uint64),
                ("episode_events", C.c_uint64), ("matched_pairs", C.c_uint64),
                ("tile_steps", C.c_uint64), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("pass1_ms", C.c_double), ("pass2_ms", C.c_double), ("map_ms", C.c_double),
                ("concat_ms", C.c_double), ("total_ms", C.c_double),
                ("bound_words", C.c_uint64), ("bound_ms", C.c_double),
                ("chain_launches", C.c_uint64), ("items_tracked", C.c_uint64),
                ("sort_fallbacks", C.c_uint64)]

    _names = None

    def as_dict(self) -> dict:
        names = Stats._names or [name for name, _ in self._fields_]
        Stats._names = names
        return {name: getattr(self, name) for name in names}


class MineConfig(C.Structure):
    _fields_ = [("threshold", C.c_uint64), ("max_level", C.c_uint64), ("alpha_low", i64p),
                ("alpha_high", i64p), ("n_alpha", C.c_uint64), ("mode", C.c_uint32)]


class EpisodeBatchOut(C.Structure):
    """EpisodeBatch as written by the library (raw addresses: cheap to copy out)."""
    _fields_ = [("n_episodes", C.c_uint64), ("offsets", C.c_void_p), ("types", C.c_void_p),
                ("low", C.c_void_p), ("high", C.c_void_p)]


class MineResultOut(C.Structure):
    """epi_mine_result with raw-address fields (same layout as MineResult)."""
    _fields_ = [("n_levels", C.c_uint64), ("level_candidates", C.c_void_p), ("level_offsets", C.c_void_p),
                ("level_ms", C.c_void_p), ("frequent", EpisodeBatchOut), ("counts", C.c_void_p),
                ("totals", Stats)]


def copy_addr(addr, count: int, dtype) -> np.ndarray:
    """Copy `count` elements at a library-owned address into a new array."""
    if not count:
        return np.zeros(0, dtype=dtype)
    dt = np.dtype(dtype)
    return np.frombuffer((C.c_char * (count * dt.itemsize)).from_address(addr), dtype=dt).copy()


class MineResult(C.Structure):
    _fields_ = [("n_levels", C.c_uint64), ("level_candidates", u64p), ("level_offsets", u64p),
                ("level_ms", f64p), ("frequent", EpisodeBatch), ("counts", u64p),
                ("totals", Stats)]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)


class Shard(C.Structure):
    _fields_ = [("rank", C.c_uint32), ("world", C.c_uint32), ("min_shard", C.c_uint64),
                ("allgather", ALLGATHER_FN), ("user", C.c_void_p)]


# Symbols every build must export (checked by the CPU test-suite).
EXPORTS = ("epi_create", "epi_destroy", "epi_last_error", "epi_status_name", "epi_load_stream",
           "epi_load_stream_device", "epi_stream_size", "epi_count", "epi_mine", "epi_generate",
           "epi_free", "epi_generate_candidates", "epi_version", "epi_probe_int32",
           "epi_generate_bursty", "epi_find_occurrences", "epi_count_tracking", "epi_parse_events",
           "epi_mine_sharded", "epi_count_sharded", "epi_write_events", "epi_read_events",
           "epi_load_stream_file", "epi_random_episodes", "epi_count_mapconcat", "epi_create_multi",
           "epi_world", "epi_uses_nccl", "epi_stream_upload_bytes", "epi_generate_stream",
           "epi_stream_download", "epi_generate_bursty_stream")


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"episodic_b200 native library not built: {LIB_PATH} is missing "
            "(run __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    sig = {
        "epi_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
        "epi_create_multi": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p)]),
        "epi_world": (C.c_uint32, [C.c_void_p]),
        "epi_stream_upload_bytes": (C.c_uint64, [C.c_void_p]),
        "epi_uses_nccl": (C.c_int, [C.c_void_p]),
        "epi_destroy": (None, [C.c_void_p]),
        "epi_last_error": (C.c_char_p, [C.c_void_p]),
        "epi_status_name": (C.c_char_p, [C.c_int]),
        "epi_load_stream": (C.c_int, [C.c_void_p, u32p, i64p, C.c_uint64, C.c_uint32]),
        "epi_load_stream_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32]),
        "epi_stream_size": (C.c_uint64, [C.c_void_p]),
        "epi_count": (C.c_int, [C.c_void_p, C.POINTER(EpisodeBatch), C.c_uint64, C.c_uint32, u64p, u8p,
                                C.POINTER(Stats)]),
        "epi_mine": (C.c_int, [C.c_void_p, C.POINTER(MineConfig), C.POINTER(MineResultOut)]),
        "epi_mine_sharded": (C.c_int, [C.c_void_p, C.POINTER(MineConfig), C.POINTER(Shard),
                                       C.POINTER(MineResultOut)]),
        "epi_count_sharded": (C.c_int, [C.c_void_p, C.POINTER(EpisodeBatch), C.c_uint64, C.c_uint32,
                                        C.POINTER(Shard), u64p, u8p, C.POINTER(Stats)]),
        "epi_write_events": (C.c_int, [C.c_char_p, u32p, i64p, C.c_uint64, C.c_uint32]),
        "epi_read_events": (C.c_int, [C.c_char_p, C.POINTER(u32p), C.POINTER(i64p), u64p,
                                      C.POINTER(C.c_uint32)]),
        "epi_load_stream_file": (C.c_int, [C.c_void_p, C.c_char_p]),
        "epi_parse_events": (C.c_int, [C.c_char_p, C.c_uint64, C.POINTER(u32p), C.POINTER(i64p), u64p,
                                       C.POINTER(C.c_void_p), C.POINTER(C.c_uint32)]),
        "epi_find_occurrences": (C.c_int, [C.c_void_p, C.POINTER(EpisodeBatch), C.c_uint32,
                                           C.POINTER(u64p), C.POINTER(i64p), C.POINTER(i64p)]),
        "epi_count_tracking": (C.c_int, [C.c_void_p, C.POINTER(EpisodeBatch), C.c_uint32, u64p,
                                         C.POINTER(Stats)]),
        "epi_count_mapconcat": (C.c_int, [C.c_void_p, C.POINTER(EpisodeBatch), C.c_uint64, u64p,
                                          C.POINTER(Stats)]),
        "epi_generate": (C.c_int, [C.c_uint32, C.c_double, C.c_double, C.c_uint64,
                                   C.POINTER(EpisodeBatch), f64p, C.POINTER(u32p), C.POINTER(i64p),
                                   u64p]),
        "epi_free": (None, [C.c_void_p]),
        "epi_generate_stream": (C.c_int, [C.c_void_p, C.c_uint32, C.c_double, C.c_double, C.c_uint64,
                                          C.POINTER(EpisodeBatch), f64p]),
        "epi_stream_download": (C.c_int, [C.c_void_p, u32p, i64p]),
        "epi_generate_bursty_stream": (C.c_int, [C.c_void_p, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                                 C.c_double, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                                 C.POINTER(EpisodeBatch), f64p]),
        "epi_generate_bursty": (C.c_int, [C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_double,
                                          C.c_double, C.c_double, C.c_double, C.c_uint64,
                                          C.POINTER(EpisodeBatch), f64p, C.POINTER(u32p),
                                          C.POINTER(i64p), u64p]),
        "epi_generate_candidates": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(EpisodeBatch), i64p, i64p,
                                              C.c_uint64, C.c_uint32, C.POINTER(EpisodeBatch)]),
        "epi_random_episodes": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                          u32p, u32p]),
        "epi_version": (C.c_char_p, []),
        "epi_probe_int32": (C.c_int, [C.c_int, C.c_int, f64p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def copy_out(p, count: int, dtype) -> np.ndarray:
    """Copy `count` elements from a library-owned pointer into a new array
    (memmove: no per-call ctypes array type as with np.ctypeslib.as_array)."""
    out = np.empty(count, dtype=dtype)
    if count:
        C.memmove(out.ctypes.data, p, count * out.itemsize)
    return out


class CSR:
    """Episode batch in the C-ABI's CSR layout, kept alive with its arrays."""

    def __init__(self, offsets, types, low, high):
        self.offsets = np.ascontiguousarray(offsets, dtype=np.uint32)
        self.types = np.ascontiguousarray(types, dtype=np.uint32)
        self.low = np.ascontiguousarray(low, dtype=np.int64)
        self.high = np.ascontiguousarray(high, dtype=np.int64)
        self._struct = None

    @property
    def struct(self) -> EpisodeBatch:
        """The C-ABI view (built on first use; it borrows this object's arrays)."""
        if self._struct is None:
            self._struct = EpisodeBatch(len(self.offsets) - 1, ptr(self.offsets, C.c_uint32),
                                        ptr(self.types, C.c_uint32), ptr(self.low, C.c_int64),
                                        ptr(self.high, C.c_int64))
        return self._struct

    def __len__(self):
        return len(self.offsets) - 1

    @staticmethod
    def from_struct(b: EpisodeBatch) -> "CSR":
        n = int(b.n_episodes)
        if n == 0:
            return CSR(np.zeros(1, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.int64),
                       np.zeros(0, np.int64))
        off = copy_out(b.offsets, n + 1, np.uint32)
        nt = int(off[-1])
        nc = nt - n
        return CSR(off, copy_out(b.types, nt, np.uint32), copy_out(b.low, nc, np.int64),
                   copy_out(b.high, nc, np.int64))

    def episode(self, e: int):
        b, en = int(self.offsets[e]), int(self.offsets[e + 1])
        cb = b - e
        return ([int(x) for x in self.types[b:en]],
                [(int(self.low[cb + k]), int(self.high[cb + k])) for k in range(en - b - 1)])
