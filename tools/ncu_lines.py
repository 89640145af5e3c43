"""Per-source-line warp-stall samples from an ncu report (--import-source, -lineinfo builds).

  python tools/ncu_lines.py REPORT.ncu-rep [--top 40] [--file tqr_device.cuh]
Aggregates the cuda,sass source page: samples per (file, line), with the top stall reasons.
"""
import argparse
import collections
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--file", default="")
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, hdr = None, None
tot = collections.Counter()
why = collections.defaultdict(collections.Counter)
src = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    line = int(r[0])
    try:
        n = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    key = (cur_file, line)
    tot[key] += n
    src[key] = r[1].strip()[:90]
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and r[i] not in ("", "0"):
            try:
                why[key][h[6:]] += int(r[i])
            except ValueError:
                pass
allsum = sum(tot.values()) or 1
print(f"total samples {allsum}")
for key, n in tot.most_common():
    if a.file and key[0] != a.file:
        continue
    if a.top <= 0:
        break
    a.top -= 1
    w = ", ".join(f"{k} {v}" for k, v in why[key].most_common(3))
    print(f"{100 * n / allsum:5.1f}%  {key[0]}:{key[1]:<5} {src[key]:<90} [{w}]")
