"""Event-file ingest (load_stream, E/io.hpp:22-67) through the native
multi-threaded parser (csrc/io.cpp, epi_parse_events). No GPU needed.

Cases follow the reference's own tests (T/test_core.cpp:76-127): comments
and CRLF, empty input, regression / bad time / missing comma with the line
number, serialize -> load round trips. Fuzzed texts and a multi-chunk file
(> 1 MiB, so the parallel path runs) are compared with the reference's
load_stream compiled in oracle/_ref (messages and line numbers included)."""
import numpy as np
import pytest

import oracle
from instances import InstanceRng, random_stream
from paper_0905_2203_b200 import (DataError, EventStream, load_stream, load_stream_file,
                                  serialize_stream)

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def test_reads_events_comments_and_crlf():
    ls = load_stream("# neurons\nA,10\nB,18\r\n\nC,20\n")
    assert ls.stream.size() == 3
    assert [ls.stream.time_at(i) for i in range(3)] == [10, 18, 20]
    assert ls.symbols[ls.stream.type_at(1)] == "B"
    assert ls.symbols == ["A", "B", "C"] and ls.stream.alphabet_size() == 3


def test_empty_input_yields_empty_stream():
    for text in ("", "\n", "# only a comment\n\r\n"):
        ls = load_stream(text)
        assert ls.stream.size() == 0 and ls.symbols == [] and ls.stream.alphabet_size() == 0


@pytest.mark.parametrize("text,line,msg", [
    ("A,5\nA,3\n", 2, "line 2: time regression (3 after 5)"),
    ("A,5\nB,x\n", 2, "line 2: bad time 'x'"),
    ("A5\n", 1, "line 1: expected '<name>,<time_ms>'"),
    (",5\n", 1, "line 1: expected '<name>,<time_ms>'"),
    ("# c\nA,-1\n", 2, "line 2: bad time '-1'"),
    ("A,\n", 1, "line 1: bad time ''"),
    ("A,5 \n", 1, "line 1: bad time '5 '"),
    ("A,1\n\nB,99999999999999999999\n", 3, "line 3: bad time '99999999999999999999'"),
])
def test_errors_name_the_line(text, line, msg):
    with pytest.raises(DataError) as ei:
        load_stream(text)
    assert str(ei.value) == msg and ei.value.line == line


def test_name_keeps_inner_commas_and_spaces():
    ls = load_stream("a,b,1\n a ,2\na,b,3\n")
    assert ls.symbols == ["a,b", " a "]
    assert ls.stream.types().tolist() == [0, 1, 0]


def test_missing_trailing_newline_and_ties():
    ls = load_stream("x,1\ny,1\nx,2")
    assert ls.stream.types().tolist() == [0, 1, 0] and ls.stream.times().tolist() == [1, 1, 2]


def test_serialize_then_load_round_trips_random_streams():
    rng = InstanceRng(23)
    for _ in range(50):
        types, times, alphabet = random_stream(rng)
        s = EventStream.from_arrays(types, times, alphabet)
        text = serialize_stream(s)
        back = load_stream(text)
        assert back.stream.size() == s.size()
        assert back.stream.times().tolist() == list(times)
        assert [back.symbols[t] for t in back.stream.types().tolist()] == [str(t) for t in types]


def test_file_variant(tmp_path):
    p = tmp_path / "events.csv"
    p.write_bytes(b"n1,3\r\nn2,4\r\n")
    ls = load_stream_file(str(p))
    assert ls.symbols == ["n1", "n2"]
    with pytest.raises(DataError, match="cannot open event file"):
        load_stream_file(str(tmp_path / "missing.csv"))


def _random_text(rng, lines, err_rate):
    names = ["n%d" % k for k in range(rng.integers(1, 40))] + ["a,b", " s p ", "#x"[1:]]
    out, t = [], 0
    for _ in range(lines):
        r = rng.random()
        if r < 0.03:
            out.append("# comment")
        elif r < 0.05:
            out.append("")
        else:
            t += int(rng.integers(0, 4))
            tt = t
            if rng.random() < err_rate:
                tt = [t - 5, "x", "", "1.5", -1][int(rng.integers(0, 5))]
            nm = names[int(rng.integers(0, len(names)))]
            if rng.random() < err_rate / 3:
                out.append(nm.replace(",", ""))  # no comma at all
                continue
            out.append(f"{nm},{tt}")
    eol = "\r\n" if rng.random() < 0.3 else "\n"
    return (eol.join(out) + (eol if rng.random() < 0.8 else "")).encode()


def _compare_with_reference(data):
    try:
        rt, rtm, rn = oracle.ref_load_stream(data)
        ref_err = None
    except oracle.RefDataError as e:
        ref_err = (str(e), e.line)
    if ref_err is not None:
        with pytest.raises(DataError) as ei:
            load_stream(data)
        assert (str(ei.value), ei.value.line) == ref_err
        return False
    ls = load_stream(data)
    assert ls.symbols == rn
    np.testing.assert_array_equal(ls.stream.types(), rt)
    np.testing.assert_array_equal(ls.stream.times(), rtm)
    return True


@needs_ref
def test_fuzz_matches_reference_load_stream():
    rng = np.random.default_rng(7)
    ok = bad = 0
    for i in range(300):
        data = _random_text(rng, int(rng.integers(0, 60)), 0.02 if i % 2 else 0.0)
        if _compare_with_reference(data):
            ok += 1
        else:
            bad += 1
    assert ok > 100 and bad > 20


@needs_ref
@pytest.mark.parametrize("fault", [None, "early", "late", "border_regression", "bad_after_regression"])
def test_multichunk_file_matches_reference(fault):
    """> 1 MiB so the chunked parallel parser runs; faults placed in late
    chunks and at chunk borders must still report the first offending line."""
    rng = np.random.default_rng(11)
    n = 200_000
    names = np.array(["e%d" % k for k in range(300)])
    tp = rng.integers(0, 300, n)
    tm = np.cumsum(rng.integers(0, 3, n))
    lines = [f"{a},{b}" for a, b in zip(names[tp].tolist(), tm.tolist())]
    if fault == "early":
        lines[1000] = "bad line"
    elif fault == "late":
        lines[n - 10] = f"late,{tm[n - 10]}x"
        lines[n - 3] = "zzz"
    elif fault in ("border_regression", "bad_after_regression"):
        text = "\n".join(lines)
        # the regression sits exactly on the line the byte midpoint lands in
        k = text.count("\n", 0, len(text) // 2) + 1
        lines[k] = f"rx,{max(int(tm[k]) - 10, 0) if tm[k] >= 10 else 0}"
        if tm[k] < 10:
            lines[k - 1] = f"ry,{int(tm[k]) + 20}"
        if fault == "bad_after_regression":
            lines[k + 5] = "nocomma"
    data = ("\n".join(lines) + "\n").encode()
    assert len(data) > (1 << 20)
    ok = _compare_with_reference(data)
    assert ok == (fault is None)


# ---- binary event files (EPIEVT01; epi_write_events / epi_read_events) -------

def test_binary_event_file_round_trip(tmp_path):
    from paper_0905_2203_b200 import read_events_binary, write_events_binary
    rng = np.random.default_rng(7)
    for n in (0, 1, 2, 3, 1000, 12345):  # odd n exercises the padding before the times
        types = rng.integers(0, 40, n).astype(np.uint32)
        times = np.sort(rng.integers(0, 10**12, n)).astype(np.int64)
        p = tmp_path / f"s{n}.evt"
        write_events_binary(str(p), types, times, 40)
        assert p.stat().st_size == 24 + (4 * n + 7) // 8 * 8 + 8 * n
        t2, tm2, a = read_events_binary(str(p))
        assert a == 40 and np.array_equal(t2, types) and np.array_equal(tm2, times)


def test_binary_event_file_errors(tmp_path):
    from paper_0905_2203_b200 import read_events_binary, write_events_binary
    with pytest.raises(DataError, match="cannot open event file"):
        read_events_binary(str(tmp_path / "missing.evt"))
    bad = tmp_path / "text.evt"
    bad.write_bytes(b"A,1\nB,2\nC,3\nD,4\nE,5\nF,6\n")
    with pytest.raises(DataError, match="not an event file"):
        read_events_binary(str(bad))
    p = tmp_path / "cut.evt"
    write_events_binary(str(p), np.arange(10, dtype=np.uint32), np.arange(10, dtype=np.int64), 10)
    p.write_bytes(p.read_bytes()[:-1])
    with pytest.raises(DataError, match="truncated event file"):
        read_events_binary(str(p))
    with pytest.raises(DataError, match="cannot open event file"):
        write_events_binary(str(tmp_path / "no" / "dir.evt"), np.zeros(1, np.uint32), np.zeros(1, np.int64), 1)
