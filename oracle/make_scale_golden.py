"""TEST INFRASTRUCTURE ONLY — writes tests/golden/scale.json: per-candidate
counts of the REFERENCE (oracle/_ref = the unmodified headers compiled in
place; count_fsm, E/fsm.hpp:101-106, episode-parallel over all host cores)
on the full-size BASELINE streams:

  cfg3        generate(64 neurons, 7813 s, 20 Hz, seed 3) = 10,004,428 events;
              ALL 10,000 candidates (mt19937_64(5): t0,t1,t2 %64, b0,b1 %3)
  cfg4        MEA-shaped bursty stream (the product's generator: the
              reference has no burst model; the stream is pinned by its FNV),
              the first 1,000 candidates of mt19937_64(44) (5 nodes over 60
              types) + the two embedded chains
  cfg5_<n>    generate(64, n/1280 s, 20 Hz, seed 5+n) for n = 1M, 10M, 100M,
              1B; the first 1,000 candidates of mt19937_64(55) (3 nodes over
              64 types) - every cfg5 cell (1k..1M candidates) draws its
              candidates from that same sequence, so this is the seeded
              subset of each cell

Streams other than cfg4 come from the reference's own generate()
(oracle.ref_generate). Run here (needs /root/reference):

    python oracle/make_scale_golden.py [cell ...]

Cells already present in scale.json are kept unless named.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden", "scale.json")

BINS = [(0, 5), (5, 10), (10, 15)]
CFG4_CHAINS = [([0, 7, 13, 21, 33], [(5, 10), (0, 5), (10, 15), (5, 10)]),
               ([40, 41, 42, 43, 44], [(0, 5)] * 4)]


def cells():
    out = {"cfg3": {"stream": {"kind": "generate", "neurons": 64, "duration_s": 7813, "rate_hz": 20, "seed": 3},
                    "cands": {"seed": 5, "count": 10000, "nodes": 3, "alphabet": 64}, "extra": []}}
    out["cfg4"] = {"stream": {"kind": "bursty", "electrodes": 60, "duration_s": 175000, "seed": 4,
                              "embedded_rate_hz": 0.5},
                   "cands": {"seed": 44, "count": 1000, "nodes": 5, "alphabet": 60},
                   "extra": [[t, [list(c) for c in cs]] for t, cs in CFG4_CHAINS]}
    for n in (1_000_000, 10_000_000, 100_000_000, 1_000_000_000):
        out[f"cfg5_{n}"] = {"stream": {"kind": "generate", "neurons": 64, "duration_s": n / 1280, "rate_hz": 20,
                                       "seed": 5 + n},
                            "cands": {"seed": 55, "count": 1000, "nodes": 3, "alphabet": 64}, "extra": []}
    return out


def make_stream(spec):
    import oracle
    if spec["kind"] == "generate":
        return oracle.ref_generate(spec["neurons"], spec["duration_s"], spec["rate_hz"], spec["seed"])
    from paper_0905_2203_b200 import BurstConfig, Embedding, Episode, generate_bursty_arrays
    emb = [Embedding(Episode(t, cs), spec["embedded_rate_hz"]) for t, cs in CFG4_CHAINS]
    return generate_bursty_arrays(BurstConfig(electrodes=spec["electrodes"], duration_s=spec["duration_s"],
                                              seed=spec["seed"], embedded=emb))


def main(argv):
    import oracle
    have = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            have = json.load(f)
    todo = cells()
    names = argv or [k for k in todo if k not in have]
    workers = os.cpu_count() or 1
    for name in names:
        spec = todo[name]
        t0 = time.time()
        types, times = make_stream(spec["stream"])
        alphabet = spec["cands"]["alphabet"] if spec["stream"]["kind"] == "bursty" else spec["stream"]["neurons"]
        c = spec["cands"]
        eps = oracle.mt_episodes(c["seed"], c["count"], c["nodes"], c["alphabet"], BINS)
        eps += [(t, [tuple(x) for x in cs]) for t, cs in spec["extra"]]
        off, et, lo, hi = oracle.csr_arrays(eps)
        t1 = time.time()
        counts = oracle.ref_count_batch(types, times, alphabet, off, et, lo, hi, algo="fsm",
                                        workers=workers, parallel=True)
        t2 = time.time()
        entry = dict(spec)
        entry.update({"n": int(len(types)), "alphabet": int(alphabet),
                      "stream_fnv": oracle.fnv_stream(types, times, alphabet),
                      "counts": [int(x) for x in counts], "sum": int(counts.sum()),
                      "checker": f"reference count_fsm (oracle/_ref), {workers} threads, "
                                 f"{t2 - t1:.0f} s"})
        have[name] = entry
        with open(OUT + ".tmp", "w") as f:
            json.dump(have, f, separators=(",", ":"))
        os.replace(OUT + ".tmp", OUT)
        print(f"{name}: n={len(types)} cands={len(eps)} sum={entry['sum']} gen {t1 - t0:.0f} s "
              f"count {t2 - t1:.0f} s", flush=True)
        del types, times


if __name__ == "__main__":
    main(sys.argv[1:])
