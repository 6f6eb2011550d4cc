"""Extract the judged numbers from one `ncu --set full` capture into JSON.

Usage: ncu_summary.py report.ncu-rep out.json [algorithmic_bytes_per_launch]

Writes duration, DRAM read/write bytes (the roofline `traffic` figure), SM /
memory / tensor-pipe utilisation and the occupancy of every captured launch.
bench.py reads `dominant_kernel_dram_bytes_per_launch` from
profiles/ncu_summary.json for the roofline `traffic` key.
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_mem_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "usecond": 1,
         "nsecond": 1e-3, "msecond": 1e3}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for k, name in WANT.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[name] = v * SCALE.get(units[i], 1)
        d["duration_us"] = d.pop("duration", None)
        launches.append(d)
    top = launches[0]
    traffic = (top.get("dram_read") or 0) + (top.get("dram_write") or 0)
    res = {"report": rep, "launches": launches, "dominant_kernel": top["kernel"],
           "dominant_kernel_dram_bytes_per_launch": traffic}
    if alg:
        res["algorithmic_bytes_per_launch"] = alg
        res["traffic_over_algorithmic"] = traffic / alg
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "launches"}, indent=1))
    for d in launches:
        print(d)


if __name__ == "__main__":
    main()
