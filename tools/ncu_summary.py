"""Summarise an ncu report (or a launch-list CSV) into the numbers profiles/ keeps.

    python tools/ncu_summary.py report gpurun_out/prof.ncu-rep  [--alg-bytes B]
    python tools/ncu_summary.py launches gpurun_out/launches.csv
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__occupancy_limit_registers", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "lts__t_bytes.sum",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "second": 1.0}


def report(path, alg_bytes=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        rec = {"kernel": vals[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    rec[m] = float(vals[i].replace(",", ""))
                except ValueError:
                    rec[m] = vals[i]
                rec[m + ".unit"] = units[i]
        rb = rec.get("dram__bytes_read.sum", 0) * SCALE.get(rec.get("dram__bytes_read.sum.unit", "byte"), 1)
        wb = rec.get("dram__bytes_write.sum", 0) * SCALE.get(rec.get("dram__bytes_write.sum.unit", "byte"), 1)
        rec["traffic_bytes"] = rb + wb
        t = rec.get("gpu__time_duration.sum", 0) * SCALE.get(rec.get("gpu__time_duration.sum.unit", "ns"), 1e-9)
        rec["duration_s"] = t
        if alg_bytes:
            rec["algorithmic_bytes"] = alg_bytes
            rec["traffic_over_algorithmic"] = rec["traffic_bytes"] / alg_bytes
        out.append(rec)
    return out


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    unit = None
    for r in rows[1:]:
        try:
            agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
            unit = r[ui]
        except ValueError:
            pass
    tot = sum(sum(v) for v in agg.values())
    return [{"kernel": k, "launches": len(v), "total": sum(v), "mean": sum(v) / len(v), "share": sum(v) / tot,
             "unit": unit} for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))]


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    alg = float(sys.argv[sys.argv.index("--alg-bytes") + 1]) if "--alg-bytes" in sys.argv else None
    res = report(path, alg) if kind == "report" else launches(path)
    print(json.dumps(res, indent=1))
