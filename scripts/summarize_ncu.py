"""Summarise ncu artefacts brought back in gpurun_out/ into text for profiles/.

  python scripts/summarize_ncu.py full gpurun_out/prof_cfg3.ncu-rep > profiles/rNN_...txt
  python scripts/summarize_ncu.py launches gpurun_out/launches_cfg2.csv > profiles/rNN_...txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
    "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Executed Instructions",
    "Registers Per Thread", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
    "Waves Per SM", "Theoretical Occupancy", "Achieved Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate",
    "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "No Eligible",
]
RAW = [
    "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum", "launch__registers_per_thread",
]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full(rep):
    rows = ncu_csv(["-i", rep, "--page", "details", "--csv"])
    hdr = rows[0]
    kernel = None
    print(f"# ncu --set full summary: {rep}")
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if kernel is None:
            kernel = d.get("Kernel Name")
            print(f"kernel: {kernel}")
        if d.get("Metric Name") in KEYS:
            print(f"  {d['Section Name'][:28]:28s} {d['Metric Name']:38s} {d['Metric Value']} {d.get('Metric Unit', '')}")
    raw = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
    if len(raw) >= 3:
        hdr, vals = raw[0], raw[2]
        print("raw counters:")
        for h, v in zip(hdr, vals):
            if h in RAW:
                print(f"  {h:70s} {v}")
        stalls = []
        for h, v in zip(hdr, vals):
            if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        print("warp-state samples (share):")
        for s, h in sorted(stalls, reverse=True)[:10]:
            print(f"  {h:30s} {s / tot * 100:5.1f}%")
    src = ncu_csv(["-i", rep, "--page", "source", "--csv", "--print-source=sass"])
    if len(src) > 2:
        hdr = src[1]
        ix = hdr.index("Instructions Executed")
        data = []
        for r in src[2:]:
            if len(r) > ix and r[ix].isdigit():
                data.append((int(r[ix]), r[1]))
        if data:
            mx = max(d[0] for d in data)
            loop = [d for d in data if d[0] >= 0.5 * mx]
            print(f"hot loop: {len(loop)} SASS instructions execute >= 50% of the max count "
                  f"(total executed {sum(d[0] for d in data)})")
            ops = defaultdict(int)
            for c, s in loop:
                op = s.split()[0] if not s.startswith("@") else s.split()[1]
                ops[op.split(".")[0]] += 1
            print("  opcode mix of the hot loop: " + ", ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", "")) / 1000.0
        tot[name] += v
        cnt[name] += 1
    # the roofline probes and torch's fill kernel (the bench's L2 flush between
    # timed steps) are not part of a step
    def outside(k):
        return "probe" in k or k.startswith("void at::")
    allt = sum(v for k, v in tot.items() if not outside(k)) or 1.0
    print(f"# ncu launch list (gpu__time_duration.sum, cold, serialised): {path}")
    print(f"{'us total':>10s} {'launches':>8s} {'share':>6s}  kernel")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        share = "" if outside(k) else f"{v / allt * 100:5.1f}%"
        print(f"{v:10.1f} {cnt[k]:8d} {share:>6s}  {k}")




def lines(rep, top=40):
    """Executed warp-instructions per CUDA source line (cuda,sass view)."""
    src = ncu_csv(["-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"])
    hi = next(i for i, r in enumerate(src) if "Instructions Executed" in r)
    hdr = src[hi]
    ix = hdr.index("Instructions Executed")
    per = defaultdict(int)
    cur = "?"
    total = 0
    for r in src[hi + 1:]:
        if len(r) <= ix:
            continue
        txt = r[1] if len(r) > 1 else ""
        v = r[ix].replace(",", "")
        # cuda rows carry "file:line" style text; sass rows start with an opcode
        if r[0] and not r[0].startswith("0x") and not v:
            cur = txt.strip()[:100]
            continue
        if v.isdigit():
            per[(r[0] if not r[0].startswith("0x") else "", cur)] += int(v)
            total += int(v)
    print(f"# executed warp-instructions per source line: {rep} (total {total})")
    for (k, c), v in sorted(per.items(), key=lambda x: -x[1])[:top]:
        print(f"{v:16d} {v / max(total, 1) * 100:5.1f}%  {k} {c}")


if __name__ == "__main__":
    {"full": full, "launches": launches, "lines": lines}[sys.argv[1]](sys.argv[2])
