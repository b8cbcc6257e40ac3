"""Summarise an ncu report: per-kernel key metrics and per-source-line stall share."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    print(" | ".join(f"{w.split('__')[-1]}={r[hdr.index(w)]}{units[hdr.index(w)]}" for w in want if w in hdr))
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kfilter and ":" in kfilter:
    args += ["--kernel-id", kfilter]
elif kfilter:
    args += ["-k", "regex:" + kfilter]
src = subprocess.run(args, capture_output=True, text=True).stdout
lines = collections.defaultdict(float)
files = collections.defaultdict(float)
cur = None
iS = None
for r in csv.reader(src.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        iS = r.index("Warp Stall Sampling (All Samples)")
        continue
    if iS is None or len(r) <= iS or not r[0].isdigit():
        continue
    try:
        v = float(r[iS] or 0)
    except ValueError:
        continue
    lines[(cur, int(r[0]), r[1].strip()[:100])] += v
    files[cur] += v
tot = sum(files.values()) or 1
for f, v in sorted(files.items(), key=lambda x: -x[1])[:8]:
    print(f"{100 * v / tot:5.1f}% {f}")
for k, v in sorted(lines.items(), key=lambda x: -x[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]} {k[2]}")
