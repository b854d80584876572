#!/usr/bin/env python
"""Summary of an .ncu-rep (one dict per launch): duration, DRAM bytes, L1/L2 hit rates, L2 and DRAM
throughput, active warps, registers, grid. Usage: ncu_summary.py <file.ncu-rep> [out.json]"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": ("duration_us", 1e-3),
    "dram__bytes_read.sum": ("dram_read_mb", None),
    "dram__bytes_write.sum": ("dram_write_mb", None),
    "l1tex__t_sector_hit_rate.pct": ("l1_hit_pct", 1),
    "lts__t_sector_hit_rate.pct": ("l2_hit_pct", 1),
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": ("lts_throughput_pct", 1),
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": ("dram_throughput_pct", 1),
    "sm__warps_active.avg.pct_of_peak_sustained_active": ("warps_active_pct", 1),
    "launch__registers_per_thread": ("regs", 1),
    "launch__grid_size": ("grid", 1),
}
UNIT = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
        "msecond": 1e3, "nsecond": 1e-3}


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(head)}
    res = []
    for r in rows[2:]:
        d = {"kernel": r[col["Kernel Name"]].split("(")[0][-40:]}
        for m, (name, _) in WANT.items():
            if m in col:
                v = float(r[col[m]].replace(",", ""))
                u = units[col[m]]
                if name.endswith("_mb") or name == "duration_us":
                    v *= UNIT.get(u, 1.0)
                d[name] = v
        res.append(d)
    txt = json.dumps(res, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main()
