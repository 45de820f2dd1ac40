"""Hot SASS lines of one kernel from an ncu report (warp-stall samples).
usage: python tools/ncu_sass_hot.py REPORT.ncu-rep KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"')),
           len(lines))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:end]))))
hdr = rows[0]
si = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
ex = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
body = rows[1:]
tot = sum(int(r[si] or 0) for r in body)
print(f"total samples {tot}, instructions {sum(int(r[ex] or 0) for r in body)}")
for idx, r in enumerate(body):
    s = int(r[si] or 0)
    if s * 100 >= tot * 1.0:
        top = sorted(((int(r[i] or 0), hdr[i]) for i in stall_cols), reverse=True)[:2]
        print(f"{idx:5d} {s:5d} {r[src].strip()[:60]:60s} {top}")
