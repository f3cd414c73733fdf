"""Summarise ncu reports / launch lists into profiles/ (run here, no GPU).

  python tools/ncu_summary.py launches <launches.csv>          -> share of device time per kernel
  python tools/ncu_summary.py report <rep.ncu-rep> [...]        -> key metrics per launch (JSON)
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active": "smem_pipe_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "warp_insts",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
SCALE = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3,
         "byte": 1.0, "Ghz": 1e9, "Mhz": 1e6}


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").strip()
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) / 1e3  # ns -> us
    tot = sum(v[1] for v in agg.values())
    out = [{"kernel": k, "launches": n, "us": round(t, 1), "share": round(t / tot, 4)}
           for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]
    return {"total_us": round(tot, 1), "kernels": out}


def sequence(path):
    """Every launch in order: kernel, grid, time (us) -- maps launches to layers."""
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
    out = []
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        out.append({"kernel": r[ki].split("(")[0].replace("void ", "").strip()[:90],
                    "grid": r[gi] if gi is not None else "", "us": round(float(r[vi].replace(",", "")) / 1e3, 2)})
    return out


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for m, k in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = v * SCALE.get(units[i], 1.0)
        if "dram_read" in d and "dram_write" in d:
            d["dram_traffic_bytes"] = d["dram_read"] + d["dram_write"]
        out.append(d)
    return out


if __name__ == "__main__":
    if sys.argv[1] == "sequence":
        for x in sequence(sys.argv[2]):
            print(f"{x['us']:9.2f}  {x['grid']:>16s}  {x['kernel']}")
        sys.exit(0)
    if sys.argv[1] == "launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        print(json.dumps({p: report(p) for p in sys.argv[2:]}, indent=1))
