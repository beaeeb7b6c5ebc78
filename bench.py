"""Benchmark: episode-events counted per second on B200 (BASELINE.json metric).

Default workload = the BASELINE.json metric's own configuration, configs[4]
("cfg5", the candidate-count sweep) at its largest single-GPU candidate set:
a 10M-event synthetic spike train (64 neurons at 20 Hz, the reference's
generate(), seed 5 + n) and 1,000,000 seeded random 3-node candidates over
the constraint bins {(0,5],(5,10],(10,15]} (one mt19937_64(55) stream: three
types % 64 then two bin indices % 3 per candidate), exact counts of every
candidate. One step = one epi_count of the whole candidate set. Work unit =
(candidate episode, stream event) pair.

  value  device-resident: stream already in HBM, step = epi_count of the
         candidates (host batch in, host counts out), timed with CUDA events.
  e2e    through the public C-ABI from pinned host buffers: epi_load_stream
         (12 B/event H2D + device validation/bitmap build) + epi_count every
         step.

--config cfg1|cfg2|cfg3|cfg4 and --cfg5-events/--cfg5-cands select the other
configs: cfg2 = Sym26 level-wise mining to level 4 with two-pass elimination;
cfg4 = MEA-shaped bursty stream (60 electrodes, ~100M events) x 10,002 5-node
candidates.
--impl reference times the reference's own CPU implementation (oracle/_ref =
the unmodified reference headers compiled in place) on the host cores: its
generate() for the stream, its count_tracking episode-parallel over a seeded
candidate subset (cfg2: its full mine()); nothing of this package is loaded.
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


CFG2_CHAINS = [([0, 1, 2, 3], [BINS[1]] * 3), ([4, 5, 6, 7], [BINS[0], BINS[1], BINS[2]]),
               ([8, 9, 10, 11], [BINS[2], BINS[0], BINS[1]]), ([12, 13, 14, 15], [BINS[1], BINS[2], BINS[0]])]
CFG4_CHAINS = [([0, 7, 13, 21, 33], [(5, 10), (0, 5), (10, 15), (5, 10)]), ([40, 41, 42, 43, 44], [(0, 5)] * 4)]
# seeded candidate sequences (mt19937_64(seed): per candidate `nodes` types %
# alphabet, then nodes-1 bin indices % 3): (seed, nodes, alphabet)
CAND_SEQ = {"cfg3": (5, 3, 64), "cfg4": (44, 5, 60), "cfg5": (55, 3, 64)}


def stream_spec(name, cfg5_events=10_000_000):
    """Generator parameters of a config's stream."""
    if name == "cfg1":
        return {"kind": "generate", "neurons": 26, "duration_s": 60, "rate_hz": 32, "seed": 1,
                "embedded": [([0, 1, 2, 3], [(5, 10)] * 3, 2.0)]}
    if name == "cfg2":
        return {"kind": "generate", "neurons": 26, "duration_s": 60, "rate_hz": 32, "seed": 1,
                "embedded": [(t, c, 5.0) for t, c in CFG2_CHAINS]}
    if name == "cfg3":
        return {"kind": "generate", "neurons": 64, "duration_s": 7813, "rate_hz": 20, "seed": 3, "embedded": []}
    if name == "cfg4":
        # MEA-culture-shaped: 60 electrodes, lognormal rates, network bursts,
        # two embedded 5-node chains; ~100M events (no reference counterpart)
        return {"kind": "bursty", "electrodes": 60, "duration_s": 175_000, "seed": 4,
                "embedded": [(t, c, 0.5) for t, c in CFG4_CHAINS]}
    if name == "cfg5":
        return {"kind": "generate", "neurons": 64, "duration_s": cfg5_events / (64 * 20), "rate_hz": 20,
                "seed": 5 + cfg5_events, "embedded": []}
    raise SystemExit(f"unknown config {name}")


def alphabet_of(spec):
    return spec["neurons"] if spec["kind"] == "generate" else spec["electrodes"]


def make_stream(name, cfg5_events=10_000_000):
    """(types, times, alphabet) of a config, from this package's generators
    (bit-exact restatement of the reference's generate())."""
    from paper_0905_2203_b200 import (BurstConfig, Embedding, Episode, GenConfig, generate_arrays,
                                      generate_bursty_arrays)
    sp = stream_spec(name, cfg5_events)
    emb = [Embedding(Episode(t, c), r) for t, c, r in sp["embedded"]]
    if sp["kind"] == "bursty":
        t, tm = generate_bursty_arrays(BurstConfig(electrodes=sp["electrodes"], duration_s=sp["duration_s"],
                                                   seed=sp["seed"], embedded=emb))
    else:
        t, tm = generate_arrays(GenConfig(sp["neurons"], sp["duration_s"], sp["rate_hz"], emb, sp["seed"]))
    return t, tm, alphabet_of(sp)


def cfg1_candidates():
    return [([a, b], [(5, 10)]) for a in range(26) for b in range(26)]


def count_candidates_csr(name, cfg5_cands=1_000_000):
    """The counting configs' candidate batch (this package's seeded
    generator; == oracle.mt_episodes, tests/test_gpu_scale.py)."""
    from paper_0905_2203_b200 import CSR, random_episodes_csr
    if name == "cfg1":
        return to_csr(cfg1_candidates())
    if name not in CAND_SEQ:
        raise SystemExit(f"{name} is not a counting config")
    seed, nodes, alphabet = CAND_SEQ[name]
    count = {"cfg3": 10_000, "cfg4": 10_000, "cfg5": cfg5_cands}[name]
    csr = random_episodes_csr(seed, count, nodes, alphabet, BINS)
    if name == "cfg4":
        x = to_csr(CFG4_CHAINS)
        csr = CSR(np.concatenate([csr.offsets, csr.offsets[-1] + x.offsets[1:]]),
                  np.concatenate([csr.types, x.types]), np.concatenate([csr.low, x.low]),
                  np.concatenate([csr.high, x.high]))
    return csr


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

def ref_stream(name, cfg5_events):
    """The config's stream from the REFERENCE's generate() (oracle/_ref);
    None for cfg4 (the reference has no burst model)."""
    import oracle
    sp = stream_spec(name, cfg5_events)
    if sp["kind"] != "generate":
        return None
    t, tm = oracle.ref_generate(sp["neurons"], sp["duration_s"], sp["rate_hz"], sp["seed"], sp["embedded"])
    return t, tm, alphabet_of(sp)


def ref_candidates(name, start, count):
    """Candidates [start, start+count) of a config's seeded sequence, drawn
    in pure Python (oracle.mt_episodes; no package code)."""
    import oracle
    if name == "cfg1":
        return cfg1_candidates()[start:start + count]
    seed, nodes, alphabet = CAND_SEQ[name]
    return oracle.mt_episodes(seed, start + count, nodes, alphabet, BINS)[start:]


def csr_arrays_of(eps):
    import oracle
    return oracle.csr_arrays(eps)


def sample_size(name, n_events, steps):
    """Candidates per CPU step: about 1,000 over the whole run (>= 1,000
    distinct seeded candidates when the run has enough steps), each step a
    few seconds of host work at most."""
    if name == "cfg1":
        return 676
    cores, _ = cpu_info()
    # enough episodes per step to keep every host core busy (episode-parallel),
    # ~1e10 episode-events per step at most (the reference runs ~0.5-5e9 ee/s
    # on 16 cores, slower on the longest streams)
    per_step = max(8 * cores, -(-1000 // max(steps, 1)))
    cap = max(2 * cores, int(1e10 // max(n_events, 1)))
    return min(per_step, cap, 1000)


def cpu_reference_count(types, times, alphabet, eps, cores):
    """The reference's counting path (oracle/_ref = reference headers compiled
    in place): episode-parallel count_tracking over candidates on all host
    cores, i.e. mine() with strategy_switch_level > max_level (its fastest
    configuration, SURVEY §8d "R2"). Falls back to the C port (count_fsm
    restatement, same threading) if the reference build is absent."""
    import oracle
    off, et, lo, hi = csr_arrays_of(eps)
    if oracle.ref_available():
        oracle.ref_count_batch(types, times, alphabet, off, et, lo, hi, algo="tracking", workers=cores,
                               parallel=True)
        return "reference"
    oracle.count_batch(types, times, off, et, lo, hi, threads=cores)
    return "port"


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
    ctx = Context(gpu)
    sp = stream_spec(args.config, args.cfg5_events)
    if sp["kind"] == "generate":
        # the reference's generate() run bit-exact on the device
        # (epi_generate_stream); the host copy feeds the end-to-end leg
        from paper_0905_2203_b200 import Embedding, Episode, GenConfig
        ctx.generate(GenConfig(sp["neurons"], sp["duration_s"], sp["rate_hz"],
                               [Embedding(Episode(t, c), r) for t, c, r in sp["embedded"]], sp["seed"]))
        types, times = ctx.download()
        alphabet = alphabet_of(sp)
    else:
        # cfg4's bursty MEA-shaped stream, also generated on the device
        from paper_0905_2203_b200 import BurstConfig, Embedding, Episode
        ctx.generate_bursty(BurstConfig(electrodes=sp["electrodes"], duration_s=sp["duration_s"], seed=sp["seed"],
                                        embedded=[Embedding(Episode(t, c), r) for t, c, r in sp["embedded"]]))
        types, times = ctx.download()
        alphabet = alphabet_of(sp)
    n = len(types)

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
        csr_all = count_candidates_csr(args.config, args.cfg5_cands)

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
        workload = {"workload": workload_name(args), "events": n, "candidates": len(csr_all),
                    "alphabet": alphabet}

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
    h2d = ctx.upload_bytes + int(s0["h2d_bytes"])  # the stream as it crossed PCIe + the batch
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
        chain = sum(s.get("chain_launches", 0) for s in stats)
        kname = "chain_kernel" if chain == map_launches else ("machines_kernel" if chain == 0 else
                                                               "chain_kernel+machines_kernel")
        tr, src = traffic_for(kname)
        kernels.append({"kernel": kname, "bound": "int32",
                        "model": "matched pairs (SURVEY 8d): 1 int op per (episode, event of an episode type)",
                        "achieved": round(ach, 4), "peak": round(peak_int, 3), "unit": "Tops/s",
                        "frac": round(ach / peak_int, 5) if peak_int else None,
                        "traffic": tr, "traffic_unit": "DRAM bytes per launch (ncu)", "traffic_source": src,
                        "peak_source": "epi_probe_int32 mode 1 (LOP3+IMAD, measured in this run)",
                        "pipe_util_ncu": pipes_for(kname),
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
                                                      "total_ms", "chain_launches")},
        # the work counted exactly (pass 2) as its own rate next to `value`
        # (which counts every candidate, pruned or not): on the exact-count
        # configs the two are equal; on cfg2 the difference is pass-1 pruning
        "exact_episode_events_per_s": sum(s["pass2_episodes"] for s in stats) * n / (step_ms * 1e-3),
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


def cpu_mine_step(types, times, cores):
    """The reference's full mine() on cfg2 (E/miner.hpp:114-173): tracking
    backend, episode-parallel at every level (strategy_switch_level >
    max_level, SURVEY §8d "R2"), all host cores. Returns (candidates, csv)."""
    import oracle
    csv, cands, _ = oracle.ref_mine(types, times, 26, 250, BINS, 4, switch_level=99, backend=1,
                                    workers=cores)
    return sum(cands), csv


def cpu_leg(args, types, times, alphabet, steps):
    """Times the reference CPU path over `steps` bounded samples of the
    workload; returns (value, seconds, sample description, kind)."""
    cores, _ = cpu_info()
    n = len(types)
    if args.config == "cfg2":
        units, secs = 0, 0.0
        for _ in range(steps):
            t0 = time.perf_counter()
            c, _ = cpu_mine_step(types, times, cores)
            secs += time.perf_counter() - t0
            units += c
        return units * n / secs, secs, ("the reference's full mine() (levels 1-4, tracking, "
                                        "strategy_switch_level > max_level) per step"), "reference"
    k = sample_size(args.config, n, steps)
    units, secs, kind = 0, 0.0, None
    for s in range(steps):
        eps = ref_candidates(args.config, (s * k) % 100_000 if args.config != "cfg1" else 0, k)
        t0 = time.perf_counter()
        kind = cpu_reference_count(types, times, alphabet, eps, cores)
        secs += time.perf_counter() - t0
        units += len(eps)
    covered = min(steps * k, 100_000) if args.config != "cfg1" else 676
    sample = (f"{k} candidates per step of the config's seeded sequence (step s: candidates "
              f"[s*{k}, (s+1)*{k}), {covered} distinct over the run) x all {n} events; count_tracking "
              "episode-parallel (mine() with strategy_switch_level > max_level); rate extrapolated "
              "linearly to the whole candidate set")
    return units * n / secs, secs, sample, kind


def cpu_baseline_for(args, types, times, alphabet):
    """One bounded CPU sample (~10-60 s of host work): up to 1,000 seeded
    candidates over the whole stream, fewer on the longest streams."""
    cores, model = cpu_info()
    steps = 1
    value, secs, sample, kind = cpu_leg(args, types, times, alphabet, steps)
    return {"value": value, "unit": "episode-events/s", "cores": cores, "kind": kind,
            "sample": f"{sample}; {steps} step(s) in {secs:.1f} s", "cpu": model}


def run_reference(args):
    """--impl reference: the reference's own CPU implementation only
    (oracle/_ref: generate(), count_tracking / mine()); this package is not
    imported."""
    import oracle
    cores, model = cpu_info()
    base = {"metric": "episode-events counted/sec (device-timed)", "impl": "reference", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic", "unit": "episode-events/s"}
    if not oracle.ref_available():
        return dict(base, unavailable="oracle/_ref/libepisodic_ref.so not built (needs /root/reference)")
    st = ref_stream(args.config, args.cfg5_events)
    if st is None:
        return dict(base, unavailable="cfg4's bursty MEA-shaped stream has no reference generator")
    types, times, alphabet = st
    n = len(types)
    if args.config == "cfg2":
        cpu_leg(args, types, times, alphabet, 1)  # warm-up: one mine()
        value, secs, sample, kind = cpu_leg(args, types, times, alphabet, args.steps)
        cands = None
    else:
        k = sample_size(args.config, n, args.steps)
        cpu_reference_count(types, times, alphabet, ref_candidates(args.config, 0, min(k, 16)), cores)
        value, secs, sample, kind = cpu_leg(args, types, times, alphabet, args.steps)
        cands = {"cfg1": 676, "cfg3": 10_000, "cfg4": 10_002, "cfg5": args.cfg5_cands}[args.config]
    ms = secs / args.steps * 1e3
    cfg = {"workload": workload_name(args), "events": n, "reference_sample": sample}
    if cands:
        cfg["candidates"] = cands
    return dict(base, value=value, ms_per_step=ms, config=cfg,
                cpu_baseline={"value": value, "unit": "episode-events/s", "cores": cores, "kind": kind,
                              "sample": sample, "cpu": model},
                e2e={"value": value, "unit": "episode-events/s", "h2d_bytes_per_step": 0,
                     "d2h_bytes_per_step": 0},
                native_so_loaded=loaded_native_libs())


def loaded_native_libs():
    try:
        with open("/proc/self/maps") as f:
            return sorted({ln.split()[-1] for ln in f if ln.rstrip().endswith(".so") and ROOT in ln})
    except OSError:
        return []


def workload_name(args):
    if args.config == "cfg2":
        return "cfg2: Sym26 mining to level 4, 3 bins, threshold 250, two-pass"
    if args.config == "cfg5":
        return (f"cfg5 cell: {args.cfg5_events} events x {args.cfg5_cands} seeded 3-node candidates, "
                "exact counts")
    return {"cfg1": "cfg1: Sym26, all 676 2-node candidates, exact counts",
            "cfg3": "cfg3: 10M events x 10,000 seeded 3-node candidates, exact counts",
            "cfg4": "cfg4: MEA-shaped ~100M bursty events x 10,002 5-node candidates, exact counts"}[args.config]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--cfg5-events", type=int, default=10_000_000, help="cfg5 cell: stream length")
    ap.add_argument("--cfg5-cands", type=int, default=1_000_000, help="cfg5 cell: 3-node candidates")
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
