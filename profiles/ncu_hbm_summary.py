"""Summarise the ncu --set full captures of profiles/ncu_hbm.sh: per kernel,
duration, DRAM bytes and throughput, achieved fraction of the measured HBM
peak, occupancy, and the busiest pipes (XU = conversions / MUFU, fp64, lsu).
Usage: ncu_hbm_summary.py dir out.json"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6551.4
M = {
    "gpu__time_duration.sum": "us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "launch__registers_per_thread": "registers",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
out = {}
for rep in sorted(glob.glob(os.path.join(sys.argv[1], "*.ncu-rep"))):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    hdr, units, r = rows[0], rows[1], rows[2]
    d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")[:90]}
    for k, name in M.items():
        if k in hdr:
            i = hdr.index(k)
            try:
                d[name] = round(float(r[i].replace(",", "")) * SCALE.get(units[i], 1), 3)
            except ValueError:
                pass
    if "us" in d and "dram_read" in d:
        d["dram_gbs"] = round((d["dram_read"] + d["dram_write"]) / d["us"] / 1e3, 1)
        d["dram_frac_of_peak"] = round(d["dram_gbs"] / PEAK, 3)
    out[os.path.basename(rep)[:-8]] = d
json.dump(out, open(sys.argv[2], "w"), indent=1)
for k, d in out.items():
    print(f"{k:18s} {d.get('us', 0):7.1f}us dram {d.get('dram_gbs', 0):7.0f} GB/s ({d.get('dram_frac_of_peak', 0):.2f}) "
          f"occ {d.get('occupancy_pct', 0):4.0f}% issue {d.get('issue_pct', 0):4.0f}% xu {d.get('xu_pct', 0):4.0f}% "
          f"fp64 {d.get('fp64_pct', 0):4.0f}% lsu {d.get('lsu_pct', 0):4.0f}%")
