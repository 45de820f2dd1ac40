#!/usr/bin/env python
"""Summarise ncu output for profiles/.

    python tools/ncu_summary.py launches <launches.csv>           # per-kernel share of device time
    python tools/ncu_summary.py full <report.ncu-rep> [config]    # key metrics per profiled launch;
                                                                  # updates profiles/ncu_traffic.json
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    m = re.search(r"(k_[a-z0-9_]+)(<[^>]*>)?", name)
    return m.group(0) if m else name.split("(")[0][-60:]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1.0, "nsecond": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6}.get(r[ui], 1.0)
        agg[short(r[ki])].append(v)
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | avg (us) | total (ms) | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / 1e6:.3f} | "
                   f"{sum(v) / tot:.3f} |")
    return "\n".join(out)


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "l1tex__t_sector_hit_rate.pct",
           "lts__t_sector_hit_rate.pct"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def full(path, config=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        rec = {"kernel": short(r[h.index("Kernel Name")])}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                rec[m] = f"{r[i]} {units[i]}".strip()
                if m.startswith("dram__bytes"):
                    try:
                        rec[m + "_bytes"] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                    except ValueError:
                        pass
        recs.append(rec)
    if config:
        tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        data = json.load(open(tj)) if os.path.exists(tj) else {}
        per = collections.defaultdict(list)
        for rec in recs:
            b = rec.get("dram__bytes_read.sum_bytes", 0) + rec.get("dram__bytes_write.sum_bytes", 0)
            per[rec["kernel"].split("<")[0]].append(b)
        data.setdefault(config, {}).update({k: sum(v) / len(v) for k, v in per.items()})
        json.dump(data, open(tj, "w"), indent=1, sort_keys=True)
    return json.dumps(recs, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        print(full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None))
