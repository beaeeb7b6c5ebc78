"""Loader measurement (HBM bounds the loader): one JSON line per
stream size with
  * the device-only loader (epi_load_stream_device: validation, gap scan,
    bitmap build; the SoA already in HBM), timed with CUDA events, its
    algorithmic HBM bytes per event and fraction of the measured copy
    bandwidth (MEASURED_PEAKS.json);
  * the end-to-end load from pageable and from pinned host arrays
    (epi_load_stream: encoded ingest for >= 4M events), wall-clock, with the
    bytes that crossed PCIe per event;
  * the raw 12 B/event upload (EPI_RAW_INGEST=1) for comparison.
Algorithmic loader traffic per event: validate reads 12 B (type + time),
the bitmap pass reads 12 B again and sets one bit (4 B read-modify-write of
a bitmap word, amortised below 4 B when events share words): 28 B/event
counted here; the bitmap memset and block sums are per tile / per 2048
events and not counted."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_0905_2203_b200 import Context, GenConfig, generate_arrays  # noqa: E402

ALG_BYTES = 28.0


def peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        for k, v in d.items():
            if "hbm" in k.lower() and isinstance(v, (int, float)):
                return float(v), f"MEASURED_PEAKS.json:{k}"
    except (OSError, ValueError):
        pass
    return 6521.4, "SURVEY §0 (MEASURED_PEAKS.json copy bandwidth)"


def best(f, k=3):
    ts = []
    for _ in range(k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def main():
    sizes = [int(x) for x in (sys.argv[1:] or ["10000000", "100000000", "1000000000"])]
    peak, peak_src = peak_hbm()
    ctx = Context(0)
    for n in sizes:
        types, times = generate_arrays(GenConfig(64, n / 1280, 20, [], 5 + n))
        n = len(types)
        d_t = torch.from_numpy(types.view(np.int32)).cuda()
        d_tm = torch.from_numpy(times).cuda()
        torch.cuda.synchronize()
        # device-only loader: the SoA is in HBM
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dev_ms = []
        for _ in range(4):
            ev0.record()
            ctx.load_device(d_t.data_ptr(), d_tm.data_ptr(), n, 64)
            ev1.record()
            torch.cuda.synchronize()
            dev_ms.append(ev0.elapsed_time(ev1))
        dms = min(dev_ms[1:])
        gbs = ALG_BYTES * n / (dms * 1e-3) / 1e9
        del d_t, d_tm
        torch.cuda.empty_cache()
        pin_t = torch.from_numpy(types).pin_memory().numpy()
        pin_tm = torch.from_numpy(times).pin_memory().numpy()
        t_page = best(lambda: ctx.load_arrays(types, times, 64))
        up_enc = ctx.upload_bytes
        t_pin = best(lambda: ctx.load_arrays(pin_t, pin_tm, 64))
        os.environ["EPI_RAW_INGEST"] = "1"
        t_raw = best(lambda: ctx.load_arrays(pin_t, pin_tm, 64))
        up_raw = ctx.upload_bytes
        del os.environ["EPI_RAW_INGEST"]
        print(json.dumps({
            "events": n,
            "device_loader": {"ms": round(dms, 3), "alg_bytes_per_event": ALG_BYTES,
                              "achieved_GBps": round(gbs, 1), "peak_GBps": peak, "peak_source": peak_src,
                              "hbm_frac": round(gbs / peak, 4)},
            "e2e_pageable": {"ms": round(t_page * 1e3, 2), "pcie_bytes_per_event": round(up_enc / n, 3)},
            "e2e_pinned": {"ms": round(t_pin * 1e3, 2), "pcie_bytes_per_event": round(up_enc / n, 3),
                           "events_per_s": n / t_pin},
            "raw_pinned_12B": {"ms": round(t_raw * 1e3, 2), "pcie_bytes_per_event": round(up_raw / n, 3),
                               "GBps": round(up_raw / t_raw / 1e9, 1)},
            "host_cores": os.cpu_count(),
        }), flush=True)
        del pin_t, pin_tm


if __name__ == "__main__":
    main()
