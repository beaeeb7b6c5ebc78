"""TEST INFRASTRUCTURE ONLY — the parity checker.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package. The product (paper_0905_2203_b200) never does.

Two checkers:
  * port  — oracle/_build/libepisodic_oracle.so, a plain-C restatement of
            count_fsm / oracle_count (E/fsm.hpp:45-106, E/oracle.hpp:21-85);
  * ref   — oracle/_ref/libepisodic_ref.so, the UNMODIFIED reference headers
            compiled in place (oracle/Makefile `ref`), when present.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(_HERE, "_build", "libepisodic_oracle.so")
REF_PATH = os.path.join(_HERE, "_ref", "libepisodic_ref.so")
U64_MAX = (1 << 64) - 1

u32p = C.POINTER(C.c_uint32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


_port = None
_ref = None


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_PATH):
            raise ImportError(f"oracle port not built: {PORT_PATH} (make -C oracle)")
        lib = C.CDLL(PORT_PATH)
        lib.orc_count_fsm.restype = C.c_uint64
        lib.orc_count_fsm.argtypes = [u32p, i64p, C.c_uint64, u32p, i64p, i64p, C.c_uint32]
        lib.orc_oracle_count.restype = C.c_uint64
        lib.orc_oracle_count.argtypes = [u32p, i64p, C.c_uint64, u32p, i64p, i64p, C.c_uint32]
        lib.orc_max_nonoverlap.restype = C.c_uint64
        lib.orc_max_nonoverlap.argtypes = [i64p, i64p, C.c_uint64]
        lib.orc_count_batch.restype = C.c_int
        lib.orc_count_batch.argtypes = [u32p, i64p, C.c_uint64, u32p, u32p, i64p, i64p, C.c_uint64,
                                        C.c_uint, u64p]
        lib.orc_validate_stream.restype = C.c_int
        lib.orc_validate_stream.argtypes = [u32p, i64p, C.c_uint64, C.c_uint32, C.c_char_p, C.c_size_t]
        lib.orc_fnv_stream.restype = C.c_uint64
        lib.orc_fnv_stream.argtypes = [u32p, i64p, C.c_uint64, C.c_uint32]
        _port = lib
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise ImportError(f"reference build missing: {REF_PATH} (make -C oracle ref)")
        lib = C.CDLL(REF_PATH)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_count_batch.restype = C.c_int
        lib.ref_count_batch.argtypes = [u32p, i64p, C.c_uint64, C.c_uint32, u32p, u32p, i64p, i64p,
                                        C.c_uint64, C.c_int, C.c_uint, C.c_int, C.c_uint64, u64p]
        lib.ref_mine.restype = C.c_int
        lib.ref_mine.argtypes = [u32p, i64p, C.c_uint64, C.c_uint32, C.c_uint64, i64p, i64p,
                                 C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_uint,
                                 C.POINTER(C.c_char_p), u64p, C.c_uint64, u64p,
                                 C.POINTER(C.c_double)]
        lib.ref_generate.restype = C.c_int
        lib.ref_generate.argtypes = [C.c_uint32, C.c_double, C.c_double, C.c_uint64, u32p, u32p, i64p,
                                     i64p, C.POINTER(C.c_double), C.c_uint64, C.POINTER(u32p),
                                     C.POINTER(i64p), u64p]
        lib.ref_free.argtypes = [C.c_void_p]
        lib.ref_find_occurrences.restype = C.c_int
        lib.ref_find_occurrences.argtypes = [u32p, i64p, C.c_uint64, C.c_uint32, u32p, u32p, i64p, i64p,
                                             C.c_int, C.POINTER(i64p), C.POINTER(i64p), u64p]
        lib.ref_default_workers.restype = C.c_uint
        lib.ref_load_stream.restype = C.c_int
        lib.ref_load_stream.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(u32p), C.POINTER(i64p), u64p,
                                        C.POINTER(C.c_void_p), C.POINTER(C.c_uint32), u64p]
        _ref = lib
    return _ref


# ---------------------------------------------------------------- port ----

def count_fsm(types, times, ep_types, low, high) -> int:
    t, tm = _u32(types), _i64(times)
    et, lo, hi = _u32(ep_types), _i64(low), _i64(high)
    return int(port().orc_count_fsm(_p(t, C.c_uint32), _p(tm, C.c_int64), len(t), _p(et, C.c_uint32),
                                    _p(lo, C.c_int64), _p(hi, C.c_int64), len(et)))


def oracle_count(types, times, ep_types, low, high) -> int:
    t, tm = _u32(types), _i64(times)
    et, lo, hi = _u32(ep_types), _i64(low), _i64(high)
    return int(port().orc_oracle_count(_p(t, C.c_uint32), _p(tm, C.c_int64), len(t),
                                       _p(et, C.c_uint32), _p(lo, C.c_int64), _p(hi, C.c_int64),
                                       len(et)))


def max_nonoverlap(intervals) -> int:
    s = _i64([a for a, _ in intervals])
    e = _i64([b for _, b in intervals])
    return int(port().orc_max_nonoverlap(_p(s, C.c_int64), _p(e, C.c_int64), len(s)))


def count_batch(types, times, offsets, ep_types, low, high, threads: int = 1) -> np.ndarray:
    t, tm = _u32(types), _i64(times)
    off, et, lo, hi = _u32(offsets), _u32(ep_types), _i64(low), _i64(high)
    n = len(off) - 1
    out = np.zeros(n, dtype=np.uint64)
    st = port().orc_count_batch(_p(t, C.c_uint32), _p(tm, C.c_int64), len(t), _p(off, C.c_uint32),
                                _p(et, C.c_uint32), _p(lo, C.c_int64), _p(hi, C.c_int64), n,
                                threads, _p(out, C.c_uint64))
    if st != 0:
        raise ValueError("interval constraint requires 0 <= low < high")
    return out


def validate_stream(types, times, alphabet):
    t, tm = _u32(types), _i64(times)
    buf = C.create_string_buffer(128)
    st = port().orc_validate_stream(_p(t, C.c_uint32), _p(tm, C.c_int64), len(t), alphabet, buf, 128)
    return st, buf.value.decode()


def fnv_stream(types, times, alphabet) -> str:
    t, tm = _u32(types), _i64(times)
    return f"{int(port().orc_fnv_stream(_p(t, C.c_uint32), _p(tm, C.c_int64), len(t), alphabet)):016x}"


# ----------------------------------------------------------- reference ----

ALGO = {"fsm": 0, "tracking": 1, "mapconcat": 2, "oracle": 3, "tracking_backward": 4}


def ref_count_batch(types, times, alphabet, offsets, ep_types, low, high, algo="fsm", workers=1,
                    parallel=True, segments=4) -> np.ndarray:
    lib = ref()
    t, tm = _u32(types), _i64(times)
    off, et, lo, hi = _u32(offsets), _u32(ep_types), _i64(low), _i64(high)
    n = len(off) - 1
    out = np.zeros(n, dtype=np.uint64)
    st = lib.ref_count_batch(_p(t, C.c_uint32), _p(tm, C.c_int64), len(t), alphabet,
                             _p(off, C.c_uint32), _p(et, C.c_uint32), _p(lo, C.c_int64),
                             _p(hi, C.c_int64), n, ALGO[algo], workers, int(parallel), segments,
                             _p(out, C.c_uint64))
    if st != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return out


def ref_mine(types, times, alphabet, threshold, bins, max_level, switch_level=3, backend=1,
             workers=1):
    """mine() of the reference; returns (csv, level_candidates, level_ms)."""
    lib = ref()
    t, tm = _u32(types), _i64(times)
    lo = _i64([b[0] for b in bins])
    hi = _i64([b[1] for b in bins])
    csv = C.c_char_p()
    cands = np.zeros(64, dtype=np.uint64)
    ms = (C.c_double * 64)()
    nl = C.c_uint64()
    st = lib.ref_mine(_p(t, C.c_uint32), _p(tm, C.c_int64), len(t), alphabet, threshold,
                      _p(lo, C.c_int64), _p(hi, C.c_int64), len(bins), max_level, switch_level,
                      backend, workers, C.byref(csv), _p(cands, C.c_uint64), 64, C.byref(nl), ms)
    if st != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    text = csv.value.decode()
    lib.ref_free(C.cast(csv, C.c_void_p))
    k = int(nl.value)
    return text, [int(x) for x in cands[:k]], [float(ms[i]) for i in range(k)]


def ref_find_occurrences(types, times, alphabet, ep_types, low, high, direction=0):
    """find_occurrences of the reference for one episode -> [(start, end)]."""
    lib = ref()
    t, tm = _u32(types), _i64(times)
    et, lo, hi = _u32(ep_types), _i64(low), _i64(high)
    off = _u32([0, len(et)])
    sp, ep, n = i64p(), i64p(), C.c_uint64()
    st = lib.ref_find_occurrences(_p(t, C.c_uint32), _p(tm, C.c_int64), len(t), alphabet,
                                  _p(off, C.c_uint32), _p(et, C.c_uint32), _p(lo, C.c_int64),
                                  _p(hi, C.c_int64), direction, C.byref(sp), C.byref(ep), C.byref(n))
    if st != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    k = int(n.value)
    out = [(sp[i], ep[i]) for i in range(k)]
    lib.ref_free(C.cast(sp, C.c_void_p))
    lib.ref_free(C.cast(ep, C.c_void_p))
    return out


def ref_load_stream(data: bytes):
    """load_stream of the reference (E/io.hpp:22-56) on `data` ->
    (types, times, names) or raises RefDataError(msg, line)."""
    lib = ref()
    tp, tm, n, nm = u32p(), i64p(), C.c_uint64(), C.c_void_p()
    alpha, line = C.c_uint32(), C.c_uint64()
    st = lib.ref_load_stream(data, len(data), C.byref(tp), C.byref(tm), C.byref(n), C.byref(nm),
                             C.byref(alpha), C.byref(line))
    if st != 0:
        raise RefDataError(lib.ref_last_error().decode(), int(line.value))
    k = int(n.value)
    types = np.array([tp[i] for i in range(k)], dtype=np.uint32)
    times = np.array([tm[i] for i in range(k)], dtype=np.int64)
    names = C.string_at(nm.value).decode()
    for q in (tp, tm):
        lib.ref_free(C.cast(q, C.c_void_p))
    lib.ref_free(nm)
    return types, times, (names.split("\n") if alpha.value else [])


class RefDataError(RuntimeError):
    def __init__(self, msg, line):
        super().__init__(msg)
        self.line = line


def ref_default_workers() -> int:
    return int(ref().ref_default_workers())


def ref_generate(neurons, duration_s, base_rate_hz, seed, embedded=()):
    """generate() of the reference (E/datagen.hpp:71-122) -> (types u32,
    times i64). `embedded`: [(types, [(lo, hi), ...], rate_hz), ...]."""
    lib = ref()
    off = _u32(np.cumsum([0] + [len(t) for t, _, _ in embedded]))
    et = _u32([x for t, _, _ in embedded for x in t] or [0])
    lo = _i64([c[0] for _, cs, _ in embedded for c in cs] or [0])
    hi = _i64([c[1] for _, cs, _ in embedded for c in cs] or [0])
    rates = np.ascontiguousarray([r for _, _, r in embedded] or [0.0], dtype=np.float64)
    tp, tm, n = u32p(), i64p(), C.c_uint64()
    st = lib.ref_generate(int(neurons), float(duration_s), float(base_rate_hz), int(seed) & U64_MAX,
                          _p(off, C.c_uint32), _p(et, C.c_uint32), _p(lo, C.c_int64), _p(hi, C.c_int64),
                          _p(rates, C.c_double), len(embedded), C.byref(tp), C.byref(tm), C.byref(n))
    if st != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    k = int(n.value)
    types = np.ctypeslib.as_array(tp, shape=(max(k, 1),))[:k].copy()
    times = np.ctypeslib.as_array(tm, shape=(max(k, 1),))[:k].copy()
    lib.ref_free(C.cast(tp, C.c_void_p))
    lib.ref_free(C.cast(tm, C.c_void_p))
    return types, times


def mt_episodes(seed, count, nodes, alphabet, bins):
    """Seeded synthetic candidates in the bench's draw order (one
    std::mt19937_64 stream: per episode `nodes` types % alphabet, then nodes-1
    bin indices % len(bins)); pure Python, for small counts."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(_HERE), "tests"))
    from instances import MT19937_64
    g = MT19937_64(seed)
    out = []
    for _ in range(count):
        t = [g() % alphabet for _ in range(nodes)]
        b = [bins[g() % len(bins)] for _ in range(nodes - 1)]
        out.append((t, b))
    return out


def csr_arrays(episodes):
    """[(types, [(lo, hi)])] -> (offsets u32, types u32, low i64, high i64)."""
    off = _u32(np.cumsum([0] + [len(t) for t, _ in episodes]))
    et = _u32([x for t, _ in episodes for x in t])
    lo = _i64([c[0] for _, cs in episodes for c in cs])
    hi = _i64([c[1] for _, cs in episodes for c in cs])
    return off, et, lo, hi
