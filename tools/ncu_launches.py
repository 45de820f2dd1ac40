"""Per-kernel summary of an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv:
launches, mean duration, share of device time, DRAM bytes per launch and the
resulting DRAM bandwidth (cold-cache, serialised replay: compare shares).
    python tools/ncu_launches.py launches.csv > summary.md"""
import collections
import csv
import re
import sys


def short(name):
    m = re.search(r"(k_[a-z0-9_]+)(<[^>]*>)?", name)
    return m.group(0) if m else name.split("(")[0][-60:]


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    idi, ki, mi, vi, ui = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value",
                                                "Metric Unit"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        if r[mi] == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1e-3)
        elif r[mi].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        per[r[idi]][r[mi]] = v
        names[r[idi]] = short(r[ki])
    agg = collections.OrderedDict()
    for i, m in per.items():
        a = agg.setdefault(names[i], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print("| kernel | launches | mean (us) | share | DRAM MB / launch | DRAM GB/s |")
    print("|---|---|---|---|---|---|")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        if t / tot < 0.001:
            continue
        print(f"| {k} | {n} | {t / n:.2f} | {t / tot:.3f} | {b / n / 1e6:.2f} | {b / t / 1e3:.0f} |")


if __name__ == "__main__":
    main(sys.argv[1])
