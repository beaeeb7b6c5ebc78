"""Per-launch DRAM traffic of the bench configs' dominant kernels from the
committed ncu captures -> profiles/roofline_traffic.json (read by bench.py)."""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

# entries whose capture is not in gpurun_out/ keep their committed values
try:
    out = json.load(open("profiles/roofline_traffic.json"))
except (OSError, ValueError):
    out = {}
CAPTURES = [
    ("cfg2:machines_kernel", "gpurun_out/prof_cfg2.ncu-rep", "profiles/r01_cfg2_machines_kernel_ncu.txt"),
    ("cfg2:bound_kernel", "gpurun_out/prof_bound.ncu-rep", "profiles/r01_cfg2_bound_kernel_ncu.txt"),
    ("cfg3:machines_kernel", "gpurun_out/prof_cfg3.ncu-rep", "profiles/r01_cfg3_machines_kernel_ncu.txt"),
    ("cfg5:chain_kernel", "gpurun_out/r02_prof_chain_default.ncu-rep", "profiles/r02_cfg5_chain_kernel_ncu.txt"),
    ("cfg3:chain_kernel", "gpurun_out/r02_prof_chain_cfg3.ncu-rep", "profiles/r02_cfg3_chain_kernel_ncu.txt"),
]
for cfg, rep, summary in CAPTURES:
    try:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units, vals = rows[0], rows[1], rows[2]
        col = {h: (u, v) for h, u, v in zip(hdr, units, vals)}

        def nbytes(name):
            u, v = col[name]
            return float(v.replace(",", "")) * SCALE[u]
        def pct(name):
            try:
                return round(float(col[name][1].replace(",", "")) / 100.0, 4)
            except (KeyError, ValueError):
                return None
        out[cfg] = {"kernel": col.get("Kernel Name", ("", ""))[1],
                    "dram_bytes_per_launch": nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum"),
                    # issue utilisation of the integer pipes (fraction of peak, ncu)
                    "pipe_util": {k: pct(f"sm__inst_executed_pipe_{k}.avg.pct_of_peak_sustained_active")
                                  for k in ("alu", "fma", "xu", "lsu")},
                    "source": summary}
    except Exception as e:  # capture missing
        print(cfg, "skipped:", e, file=sys.stderr)
json.dump(out, open("profiles/roofline_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
