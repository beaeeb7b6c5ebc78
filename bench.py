"""Benchmark: episode-events counted per second on B200 (BASELINE.json metric).

Default workload = BASELINE.json configs[1] ("cfg2"): Sym26 synthetic spike
train (26 neurons, 60 s, 32 Hz, seed 1, four embedded 4-node chains at 5 Hz:
54,750 events), level-wise mining to 4-node episodes over the constraint
alphabet {(0,5],(5,10],(10,15]} at threshold 250 with two-pass elimination.
One step = one full mine() (levels 1-4: 26 + 2,028 + 142,228 + 4
candidates). Work unit = (candidate episode, stream event) pair, counted for
every generated candidate, pruned or not (the reference counts them all).

  value  device-resident: stream already in HBM, step = epi_mine on it,
         timed with CUDA events (synchronous call; host candidate generation
         is inside the step).
  e2e    through the public C-ABI from pinned host buffers: epi_load_stream
         (12 B/event H2D + device validation/bitmap build) + epi_mine (which
         returns counts to the host) every step.

--config cfg1|cfg3|cfg4|cfg5 selects the other single-GPU configs (exact
counting only): cfg4 = MEA-shaped bursty stream (60 electrodes, ~100M
events) x 10,002 5-node candidates; cfg5 = one cell of the sweep
(--cfg5-events, --cfg5-cands: 64 types at 20 Hz, random 3-node candidates).
--impl reference times the reference's own CPU implementation (oracle/_ref,
compiled from /root/reference) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BINS = [(0, 5), (5, 10), (10, 15)]


def make_config(name):
    from paper_0905_2203_b200 import Embedding, Episode, GenConfig
    if name in ("cfg1",):
        return GenConfig(26, 60, 32, [Embedding(Episode([0, 1, 2, 3], [(5, 10)] * 3), 2.0)], 1)
    if name == "cfg2":
        eps = [([0, 1, 2, 3], [BINS[1]] * 3), ([4, 5, 6, 7], [BINS[0], BINS[1], BINS[2]]),
               ([8, 9, 10, 11], [BINS[2], BINS[0], BINS[1]]),
               ([12, 13, 14, 15], [BINS[1], BINS[2], BINS[0]])]
        return GenConfig(26, 60, 32, [Embedding(Episode(t, c), 5.0) for t, c in eps], 1)
    if name == "cfg3":
        return GenConfig(64, 7813, 20, [], 3)
    raise SystemExit(f"unknown config {name}")


def make_stream(name, cfg5_events=10_000_000):
    """(types, times, alphabet) of a bench config; synthetic, seeded."""
    from paper_0905_2203_b200 import (BurstConfig, Embedding, Episode, GenConfig, generate_arrays,
                                      generate_bursty_arrays)
    if name == "cfg4":
        # MEA-culture-shaped: 60 electrodes, lognormal
        # rates, network bursts, two embedded 5-node chains; ~100M events
        t, tm = generate_bursty_arrays(BurstConfig(electrodes=60, duration_s=175_000, seed=4,
                                                   embedded=[Embedding(c, 0.5) for c in CFG4_CHAINS()]))
        return t, tm, 60
    if name == "cfg5":
        t, tm = generate_arrays(GenConfig(64, cfg5_events / (64 * 20), 20, [], 5 + cfg5_events))
        return t, tm, 64
    t, tm = generate_arrays(make_config(name))
    return t, tm, 64 if name == "cfg3" else 26


def CFG4_CHAINS():
    from paper_0905_2203_b200 import Episode
    return [Episode([0, 7, 13, 21, 33], [(5, 10), (0, 5), (10, 15), (5, 10)]),
            Episode([40, 41, 42, 43, 44], [(0, 5)] * 4)]


def random_candidates(seed, count, alphabet, nodes):
    rng = np.random.default_rng(seed)
    return [([int(x) for x in rng.integers(0, alphabet, nodes)],
             [BINS[int(b)] for b in rng.integers(0, 3, nodes - 1)]) for _ in range(count)]


def count_candidates(name, cfg5_cands=10000):
    if name == "cfg1":
        return cfg1_candidates()
    if name == "cfg3":
        return cfg3_candidates()
    if name == "cfg4":
        return random_candidates(44, 10000, 60, 5) + [(c.types, c.constraints) for c in CFG4_CHAINS()]
    if name == "cfg5":
        return random_candidates(55, cfg5_cands, 64, 3)
    raise SystemExit(f"{name} is not a counting config")


def cfg1_candidates():
    return [([a, b], [(5, 10)]) for a in range(26) for b in range(26)]


def cfg3_candidates(count=10000):
    """mt19937_64(5): t0,t1,t2 = rng()%64 then b0,b1 = rng()%3."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from instances import MT19937_64
    g = MT19937_64(5)
    out = []
    for _ in range(count):
        t = [g() % 64 for _ in range(3)]
        b = [BINS[g() % 3] for _ in range(2)]
        out.append((t, b))
    return out


def to_csr(eps):
    from paper_0905_2203_b200 import CSR
    off = np.cumsum([0] + [len(t) for t, _ in eps]).astype(np.uint32)
    types = np.concatenate([np.asarray(t, np.uint32) for t, _ in eps])
    lo = np.array([c[0] for _, cs in eps for c in cs], np.int64)
    hi = np.array([c[1] for _, cs in eps for c in cs], np.int64)
    return CSR(off, types, lo, hi)


_NVML_CHILD = r"""
import sys, time, pynvml as p
p.nvmlInit()
bus = sys.argv[1]
h = p.nvmlDeviceGetHandleByPciBusId(bus.encode()) if ":" in bus else p.nvmlDeviceGetHandleByIndex(int(bus))
mx = p.nvmlDeviceGetMaxClockInfo(h, p.NVML_CLOCK_SM)
out = sys.stdout
while True:
    sm = p.nvmlDeviceGetClockInfo(h, p.NVML_CLOCK_SM)
    r = p.nvmlDeviceGetCurrentClocksEventReasons(h)
    out.write("%.6f %d %d %d\n" % (time.monotonic(), sm, mx, r))
    out.flush()
    time.sleep(0.0005)
"""


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region.

    NVML in a child process (about one sample per millisecond, CLOCK_MONOTONIC
    stamps filtered to the region, no GIL contention with the timed loop);
    nvidia-smi polling when NVML is unavailable."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits -> names
    BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
            0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index, bus_id=None):
        self.index = index
        self.bus_id = bus_id
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._child = None
        self._span = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def _start_child(self):
        try:
            child = subprocess.Popen([sys.executable, "-c", _NVML_CHILD, self.bus_id or str(self.index)],
                                     stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            return None
        line = child.stdout.readline()  # first sample: NVML works
        if not line:
            child.wait(timeout=5)
            return None
        self._rows = []
        self._reader = threading.Thread(target=lambda: self._rows.extend(ln.split() for ln in child.stdout),
                                        daemon=True)
        self._reader.start()
        return child

    def __enter__(self):
        self._child = self._start_child()
        if self._child is None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        self._span = [time.monotonic(), None]
        return self

    def __exit__(self, *a):
        self._span[1] = time.monotonic()
        if self._child is not None:
            time.sleep(0.002)  # a sample past the end of the region
            self._child.kill()  # the exact child started above
            self._child.wait(timeout=10)
            self._reader.join(timeout=10)
            rows = list(self._rows)
            t0, t1 = self._span
            inside = [r for r in rows if len(r) == 4 and t0 <= float(r[0]) <= t1]
            if not inside:  # region shorter than the sampling period: nearest sample
                inside = sorted((r for r in rows if len(r) == 4), key=lambda r: abs(float(r[0]) - t1))[:1]
            self.samples = [("nvml", int(r[1]), int(r[2]), int(r[3])) for r in inside]
        else:
            self._stop.set()
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        if self.samples[0][0] == "nvml":
            sm = [s[1] for s in self.samples]
            reasons = sorted({n for s in self.samples for b, n in self.BITS.items() if s[3] & b})
            return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(s[2] for s in self.samples)),
                    "reasons": reasons, "samples": len(self.samples), "source": "nvml, ~1 ms period"}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples), "source": "nvidia-smi"}


def _bus_id(gpu):
    try:
        import torch
        pr = torch.cuda.get_device_properties(gpu)
        return "%08X:%02X:%02X.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
    except Exception:
        return None


def cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return os.cpu_count() or 1, model


# ------------------------------------------------------------ CPU legs ----

def level3_sample(types, times, size, seed=11):
    """Seeded sample of the cfg2 level-3 candidates (the level that carries
    98% of the work), generated with the product's host join."""
    from paper_0905_2203_b200 import Episode, generate_candidates
    import oracle
    l1 = [Episode([t], []) for t in range(26)]
    l2 = generate_candidates(2, l1, BINS, 26)
    csr2 = to_csr([(e.types, e.constraints) for e in l2])
    c2 = oracle.count_batch(types, times, csr2.offsets, csr2.types, csr2.low, csr2.high,
                            threads=os.cpu_count() or 1)
    f2 = [e for e, c in zip(l2, c2) if c >= 250]
    l3 = generate_candidates(3, f2, BINS, 26)
    rng = np.random.default_rng(seed)
    pick = np.sort(rng.choice(len(l3), size=min(size, len(l3)), replace=False))
    return to_csr([(l3[i].types, l3[i].constraints) for i in pick]), len(l3)


def cpu_reference_rate(types, times, alphabet, csr, budget_s, min_reps=1):
    """The reference's counting path (oracle/_ref = reference headers compiled
    in place): episode-parallel count_tracking over candidates on all host
    cores, i.e. mine() with strategy_switch_level > max_level (its fastest
    configuration, SURVEY §8d "R2"). Falls back to the C port (count_fsm
    restatement, same threading) if the reference build is absent."""
    import oracle
    cores, _ = cpu_info()
    kind = "reference" if oracle.ref_available() else "port"
    reps, t_total, ee = 0, 0.0, 0
    while reps < min_reps or t_total < budget_s:
        t0 = time.perf_counter()
        if kind == "reference":
            oracle.ref_count_batch(types, times, alphabet, csr.offsets, csr.types, csr.low, csr.high,
                                   algo="tracking", workers=cores, parallel=True)
        else:
            oracle.count_batch(types, times, csr.offsets, csr.types, csr.low, csr.high, threads=cores)
        t_total += time.perf_counter() - t0
        ee += len(csr) * len(types)
        reps += 1
    return ee / t_total, kind, cores, reps, t_total


# ------------------------------------------------------------- our arm ----

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_0905_2203_b200 import Context, MODE_MINE, generate_arrays, _native

    gpu = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    # collectives on device tensors for NCCL; gloo (EPI_BENCH_BACKEND, for
    # functional runs with several ranks on one GPU) takes host tensors
    coll_dev = dev if os.environ.get("EPI_BENCH_BACKEND", "nccl") == "nccl" else None
    types, times, alphabet = make_stream(args.config, args.cfg5_events)
    n = len(types)
    ctx = Context(gpu)
    ctx.load_arrays(types, times, alphabet)

    # Pinned host copies for the end-to-end leg.
    h_types = torch.from_numpy(types).pin_memory()
    h_times = torch.from_numpy(times).pin_memory()
    ht, htm = h_types.numpy(), h_times.numpy()

    # Multi-GPU: each rank counts its episode shard; one all_gather of the
    # u64 counts per level over NCCL (paper_0905_2203_b200/shard.py).
    from paper_0905_2203_b200.shard import make_allgather
    acc = []

    def count_fn(part, threshold, mode):
        c = ctx.count_csr(part, threshold, mode)
        acc.append((len(part), ctx.last_stats))
        return c

    def merged():
        keys = acc[0][1].keys() if acc else []
        st = {k: sum(s[k] for _, s in acc) for k in keys}
        if acc:
            st["segments"] = acc[-1][1]["segments"]
        return sum(u for u, _ in acc), st

    if args.config == "cfg2":
        if world == 1:
            def step():
                cands, offs, ms, csr, counts, st = ctx.mine_raw(250, BINS, 4, MODE_MINE)
                return sum(cands), st
        else:
            # device-resident mining on every rank; each level of >= 8192
            # candidates is episode-sharded and its u64 counts all-gathered
            # on the engine's stream (NCCL; gloo host-staged for functional
            # runs of several ranks on one GPU)
            ag = make_allgather(memory="cuda" if coll_dev is not None else "staged", device=dev)

            def step():
                cands, offs, ms, csr, counts, st = ctx.mine_raw(250, BINS, 4, MODE_MINE,
                                                                shard=(rank, world, 8192, ag))
                return sum(cands) / world, st  # job units, summed over ranks below
        workload = {"workload": "cfg2: Sym26 mining to level 4, 3 bins, threshold 250, two-pass",
                    "events": n, "levels": 4, "threshold": 250, "bins": BINS}
    else:
        eps = count_candidates(args.config, args.cfg5_cands)
        csr_all = to_csr(eps)

        if world > 1:
            # epi_count_sharded: >= 4096 episodes per rank shard by episode,
            # fewer shard the MapConcatenate segments by time
            ag = make_allgather(memory="cuda" if coll_dev is not None else "staged", device=dev)

        def step():
            acc.clear()
            if world == 1:
                count_fn(csr_all, 1, 0)
                return merged()
            ctx.count_csr(csr_all, 1, 0, shard=(rank, world, 4096 * world, ag))
            return len(csr_all) / world, ctx.last_stats  # job units, summed over ranks below
        workload = {"workload": f"{args.config}: exact counts of {len(eps)} "
                                f"{len(eps[0][0])}-node candidates",
                    "events": n, "candidates": len(eps), "alphabet": alphabet}

    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, k):
        times_ms, units, stats = [], 0, []
        for _ in range(k):
            flush.zero_()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            u, st = fn()
            e1.record()
            torch.cuda.synchronize()
            times_ms.append(e0.elapsed_time(e1))
            units += u
            stats.append(st)
        return times_ms, units, stats

    for _ in range(args.warmup):
        step()
    barrier()
    with ClockSampler(gpu, _bus_id(gpu)) as clk:
        t_ms, cand_total, stats = timed(step, args.steps)
    clocks = clk.summary()
    step_ms = float(np.sum(t_ms))
    red_dev = coll_dev if coll_dev is not None else torch.device("cpu")
    if world > 1:
        tt = torch.tensor([step_ms], device=red_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        step_ms = float(tt.item())
        ct = torch.tensor([cand_total], device=red_dev, dtype=torch.float64)
        dist.all_reduce(ct)
        cand_total = float(ct.item())
    value = cand_total * n / (step_ms * 1e-3)

    # End-to-end: pinned host stream -> C-ABI load + mine/count -> host counts.
    def e2e_step():
        ctx.load_arrays(ht, htm, alphabet)
        return step()
    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    e_ms, e_units, e_stats = timed(e2e_step, args.steps)
    e_total_ms = float(np.sum(e_ms))
    if world > 1:
        tt = torch.tensor([e_total_ms], device=red_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e_total_ms = float(tt.item())
        ct = torch.tensor([e_units], device=red_dev, dtype=torch.float64)
        dist.all_reduce(ct)
        e_units = float(ct.item())
    e2e_value = e_units * n / (e_total_ms * 1e-3)
    s0 = e_stats[-1]
    h2d = n * 12 + int(s0["h2d_bytes"])
    d2h = int(s0["d2h_bytes"])

    # Roofline of the dominant kernel, per launch, from the engine's CUDA
    # events on its own stream. Two kernel families carry the device time:
    #   machines_kernel (segment-map automaton; exact counts): matched-pair
    #     model of SURVEY 8d, 1 INT32 op per (episode, event of one of its
    #     types), against the measured LOP3+IMAD issue rate;
    #   bound_kernel (pass 1, popcount bound): 1 POPC per (candidate, 32 ms
    #     tile) word pair, against the measured POPC (XU pipe) issue rate.
    map_ms = sum(s["map_ms"] for s in stats)
    map_launches = sum(s["map_launches"] for s in stats)
    matched = sum(s["matched_pairs"] for s in stats)
    tiles = sum(s["tile_steps"] for s in stats)
    bound_ms = sum(s["bound_ms"] for s in stats)
    bound_words = sum(s["bound_words"] for s in stats)
    total_dev_ms = sum(s["total_ms"] for s in stats)
    peak_int = ctypes_probe(_native, gpu, 1)
    peak_popc = ctypes_probe(_native, gpu, 2)
    traffic_all = {}
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
            traffic_all = json.load(f)
    except (OSError, ValueError):
        pass

    def traffic_for(kernel):
        tj = traffic_all.get(f"{args.config}:{kernel}") or (traffic_all.get(args.config)
                                                            if kernel == "machines_kernel" else None)
        return (tj["dram_bytes_per_launch"], tj["source"]) if tj else (None, None)

    def pipes_for(kernel):
        tj = traffic_all.get(f"{args.config}:{kernel}")
        return tj.get("pipe_util") if tj else None

    kernels = []
    if map_ms > 0:
        ach = matched / (map_ms * 1e-3) / 1e12
        tr, src = traffic_for("machines_kernel")
        kernels.append({"kernel": "machines_kernel", "bound": "int32",
                        "model": "matched pairs (SURVEY 8d): 1 int op per (episode, event of an episode type)",
                        "achieved": round(ach, 4), "peak": round(peak_int, 3), "unit": "Tops/s",
                        "frac": round(ach / peak_int, 5) if peak_int else None,
                        "traffic": tr, "traffic_unit": "DRAM bytes per launch (ncu)", "traffic_source": src,
                        "peak_source": "epi_probe_int32 mode 1 (LOP3+IMAD, measured in this run)",
                        "pipe_util_ncu": pipes_for("machines_kernel"),
                        "launches": map_launches, "avg_launch_ms": round(map_ms / max(map_launches, 1), 5),
                        "device_ms": round(map_ms, 4),
                        "share_of_device_time": round(map_ms / total_dev_ms, 4) if total_dev_ms else None,
                        "tile_steps_per_s": tiles / (map_ms * 1e-3),
                        "dense_model_ee_per_s_kernel": sum(s["episode_events"] for s in stats) / (map_ms * 1e-3)})
    if bound_ms > 0:
        ach = bound_words / (bound_ms * 1e-3) / 1e12
        tr, src = traffic_for("bound_kernel")
        kernels.append({"kernel": "bound_kernel", "bound": "int32",
                        "model": "pass-1 popcount bound: 1 POPC per (candidate, 32 ms tile) word pair",
                        "achieved": round(ach, 4), "peak": round(peak_popc, 3), "unit": "Tops/s",
                        "frac": round(ach / peak_popc, 5) if peak_popc else None,
                        "traffic": tr, "traffic_unit": "DRAM bytes per launch (ncu)", "traffic_source": src,
                        "peak_source": "epi_probe_int32 mode 2 (POPC, XU pipe, measured in this run)",
                        "pipe_util_ncu": pipes_for("bound_kernel"),
                        "device_ms": round(bound_ms, 4),
                        "share_of_device_time": round(bound_ms / total_dev_ms, 4) if total_dev_ms else None})
    kernels.sort(key=lambda k: -k["device_ms"])
    roofline = dict(kernels[0]) if kernels else {"bound": "int32", "achieved": None, "peak": None,
                                                 "unit": "Tops/s", "frac": None, "traffic": None}
    roofline["kernels"] = kernels

    out = {
        "metric": "episode-events counted/sec (device-timed)",
        "value": value, "unit": "episode-events/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": dict(workload, parallelism=f"episode-shard x{world}",
                       l2="flushed (512 MiB write) between timed steps"),
        "e2e": {"value": e2e_value, "unit": "episode-events/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e_total_ms / args.steps},
        "roofline": roofline,
        "clocks": clocks,
        "gpu_launches": int(sum(s["kernel_launches"] for s in stats)),
        "pass_breakdown": {k: stats[-1][k] for k in ("episodes", "pass1_groups", "pass2_episodes",
                                                      "pruned", "segments", "patches", "pass1_ms",
                                                      "pass2_ms", "map_ms", "concat_ms", "bound_ms",
                                                      "total_ms")},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_for(args, types, times, alphabet)
    ctx.close()
    return out


def ctypes_probe(native, device, mode=1):
    import ctypes
    v = ctypes.c_double(0)
    st = native.lib.epi_probe_int32(device, mode, ctypes.byref(v))
    return v.value if st == 0 else 0.0


def cpu_baseline_for(args, types, times, alphabet):
    cores, model = cpu_info()
    if args.config == "cfg2":
        csr, n3 = level3_sample(types, times, 20000)
        sample = (f"{len(csr)} seeded cfg2 level-3 candidates (of {n3}) x {len(types)} events, "
                  "count_tracking episode-parallel on all cores")
    elif args.config == "cfg1":
        csr = to_csr(cfg1_candidates())
        sample = f"all 676 cfg1 candidates x {len(types)} events"
    elif args.config == "cfg3":
        csr = to_csr(cfg3_candidates(64))
        sample = f"first 64 cfg3 candidates x {len(types)} events"
    else:
        k = 16 if len(types) > 50_000_000 else 64
        csr = to_csr(count_candidates(args.config, args.cfg5_cands)[:k])
        sample = f"first {k} {args.config} candidates x {len(types)} events"
    rate, kind, cores, reps, secs = cpu_reference_rate(types, times, alphabet, csr, args.cpu_seconds)
    return {"value": rate, "unit": "episode-events/s", "cores": cores, "kind": kind,
            "sample": f"{sample}; {reps} reps in {secs:.1f} s", "cpu": model}


def run_reference(args):
    types, times, alphabet = make_stream(args.config, args.cfg5_events)
    cores, model = cpu_info()
    if args.config == "cfg2":
        csr, n3 = level3_sample(types, times, 20000)
        sample = f"{len(csr)} seeded cfg2 level-3 candidates (of {n3})"
    elif args.config == "cfg1":
        csr = to_csr(cfg1_candidates())
        sample = "all 676 cfg1 candidates"
    elif args.config == "cfg3":
        csr = to_csr(cfg3_candidates(64))
        sample = "first 64 cfg3 candidates"
    else:
        k = 16 if len(types) > 50_000_000 else 64
        csr = to_csr(count_candidates(args.config, args.cfg5_cands)[:k])
        sample = f"first {k} {args.config} candidates"
    for _ in range(args.warmup):
        cpu_reference_rate(types, times, alphabet, csr, 0.0)
    rates = []
    kind = None
    t_all = 0.0
    for _ in range(args.steps):
        r, kind, cores, reps, secs = cpu_reference_rate(types, times, alphabet, csr, 0.0)
        rates.append(r)
        t_all += secs
    value = len(csr) * len(types) * args.steps / t_all
    return {"metric": "episode-events counted/sec (device-timed)", "impl": "reference",
            "value": value, "unit": "episode-events/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_all / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": f"{args.config} (reference CPU: {sample})", "events": len(types)},
            "cpu_baseline": {"value": value, "unit": "episode-events/s", "cores": cores, "kind": kind,
                             "sample": f"{sample} x {len(types)} events per step, count_tracking "
                                       "episode-parallel (mine() with strategy_switch_level > "
                                       "max_level) on all cores", "cpu": model},
            "e2e": {"value": value, "unit": "episode-events/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--cfg5-events", type=int, default=10_000_000, help="cfg5 cell: stream length")
    ap.add_argument("--cfg5-cands", type=int, default=10_000, help="cfg5 cell: 3-node candidates")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        backend = os.environ.get("EPI_BENCH_BACKEND", "nccl")
        gpu = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(gpu)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(backend)
    out = run_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
