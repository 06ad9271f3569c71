"""Summarise an ncu capture into profiles/ (committed evidence).

    python scripts/ncu_summarize.py TAG [gpurun_out/prof_TAG.ncu-rep] [gpurun_out/launches_TAG.csv]

Writes profiles/TAG_ncu_summary.md (per-kernel key metrics + launch-list
shares) and, for the dominant kernel, profiles/augment_crop_traffic.json which
bench.py reads for roofline.traffic.
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM throughput"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of ncu peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_shared_mem", "occ limit (smem)"),
    ("smsp__inst_executed.sum", "instructions"),
    ("lts__t_bytes.sum", "L2 bytes"),
]


def to_bytes(v: float, unit: str) -> float:
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def to_us(v: float, unit: str) -> float:
    return v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3,
                "ms": 1e3, "second": 1e6}.get(unit, 1)


def raw_rows(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def launches(path: str):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "")
        agg[name][0] += 1
        agg[name][1] += to_us(float(r[vi].replace(",", "")), r[ui])
    return agg


def main():
    tag = sys.argv[1]
    rep = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
    lcsv = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    md = [f"# ncu summary {tag}", "",
          f"Source: `{os.path.relpath(rep, ROOT)}` (ncu --set full --clock-control none) and "
          f"`{os.path.relpath(lcsv, ROOT)}` (gpu__time_duration.sum launch list).", ""]
    if os.path.exists(lcsv):
        agg = launches(lcsv)
        tot = sum(v[1] for v in agg.values())
        md += ["## Launch list (cold-cache, serialised: compare shares)", "",
               "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            md.append(f"| `{k}` | {v[0]} | {v[1]:.1f} | {v[1] / v[0]:.2f} | {100 * v[1] / tot:.1f}% |")
        md.append("")
    traffic = None
    if os.path.exists(rep):
        hdr, units, rows = raw_rows(rep)
        ki = hdr.index("Kernel Name")
        md += ["## Per-launch metrics (--set full)", ""]
        cols = [(m, lab) for m, lab in METRICS if m in hdr]
        md.append("| kernel | " + " | ".join(lab for _, lab in cols) + " |")
        md.append("|---|" + "---|" * len(cols))
        aug = []
        for r in rows:
            vals = []
            for m, _ in cols:
                i = hdr.index(m)
                vals.append(f"{r[i]} {units[i]}".strip())
            name = r[ki].split("(")[0].replace("(anonymous namespace)::", "")
            md.append(f"| `{name}` | " + " | ".join(vals) + " |")
            kern = ("augment_crop" if "augment_crop" in name else
                    "augment_resize" if "augment_resize" in name else None)
            if kern:
                rd = to_bytes(float(r[hdr.index("dram__bytes_read.sum")]), units[hdr.index("dram__bytes_read.sum")])
                wr = to_bytes(float(r[hdr.index("dram__bytes_write.sum")]), units[hdr.index("dram__bytes_write.sum")])
                grid = int(float(r[hdr.index("launch__grid_size")]))
                bf16 = r[ki].split("<")[1].startswith(("1", "true")) if "<" in r[ki] else False
                aug.append((rd, wr, grid, bf16, kern))
        md.append("")
        if aug:
            kern = aug[0][4]
            sel = [a for a in aug if a[4] == kern]
            rd = sum(a[0] for a in sel) / len(sel)
            wr = sum(a[1] for a in sel) / len(sel)
            # crop: 7 bands per sample; resize: 14 bands of 16 rows per sample (224 out)
            per = 7 if kern == "augment_crop" else 14
            traffic = {"kernel": kern, "tag": tag, "dram_read_bytes_per_launch": rd,
                       "dram_write_bytes_per_launch": wr, "dram_bytes_per_launch": rd + wr,
                       "grid": sel[0][2], "dtype": "bf16" if sel[0][3] else "fp32",
                       "per_gpu_batch": sel[0][2] // per if sel[0][2] % per == 0 else None,
                       "note": "writes still dirty in L2 at kernel end are not counted"}
    out_md = os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md")
    os.makedirs(os.path.dirname(out_md), exist_ok=True)
    with open(out_md, "w") as f:
        f.write("\n".join(md) + "\n")
    print(out_md)
    if traffic:
        p = os.path.join(ROOT, "profiles", f"{traffic['kernel']}_traffic.json")
        with open(p, "w") as f:
            json.dump(traffic, f, indent=1)
        print(p, traffic)


if __name__ == "__main__":
    main()
