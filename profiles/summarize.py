"""Turn ncu outputs brought back in gpurun_out/ into committed summaries.

    python profiles/summarize.py launches gpurun_out/launches.csv profiles/r01_launches.md
    python profiles/summarize.py full gpurun_out/prof_lz.ncu-rep profiles/r01_lanczos_full.md [lanczos_dram.json]
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys


def launches(csv_path, out_md):
    rows = list(csv.reader(open(csv_path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total us | share |", "|---|---:|---:|---:|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
    open(out_md, "w").write(
        "# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n\n"
        f"source: `{csv_path}`; compare shares, not absolutes\n\n" + "\n".join(lines) + "\n")
    print("\n".join(lines[:12]))


def full(rep, out_md, dram_json=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
            "smsp__inst_executed.sum", "lts__t_sectors_srcunit_tex_op_read.sum"]
    out = ["| kernel | " + " | ".join(w.split("__")[-1] for w in want) + " |",
           "|---|" + "---|" * len(want)]
    recs = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0]
        vals = [r[h.index(w)] if w in h else "-" for w in want]
        out.append(f"| {name} | " + " | ".join(vals) + " |")
        rec = {"kernel": name}
        for w, v in zip(want, vals):
            rec[w] = v
        recs.append(rec)
    units = [rows[1][h.index(w)] if w in h else "" for w in want]
    open(out_md, "w").write(f"# ncu --set full summary\n\nsource: `{rep}`\n\nunits: "
                            + ", ".join(f"{w}={u}" for w, u in zip(want, units)) + "\n\n" + "\n".join(out) + "\n")
    print("\n".join(out))
    if dram_json:
        def num(x):
            try:
                return float(str(x).replace(",", ""))
            except ValueError:
                return None
        first = recs[0]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = num(first["dram__bytes_read.sum"]) * scale.get(units[1], 1)
        wr = num(first["dram__bytes_write.sum"]) * scale.get(units[2], 1)
        json.dump({"kernel": first["kernel"], "dram_bytes_per_launch": rd + wr, "source": rep},
                  open(dram_json, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
