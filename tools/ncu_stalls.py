"""Top source lines / SASS instructions of an ncu source-page CSV with their
stall-reason breakdown: python tools/ncu_stalls.py source.csv [n]"""
import collections, csv, sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
hdr = None
cur_file = None
line_tot = collections.Counter()
line_rs = collections.defaultdict(collections.Counter)
line_src = {}
sass = []
cur_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        rs_idx = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) < 8 or r[2] == "...":
        continue
    if r[0]:          # source line
        cur_line = f"{cur_file}:{r[0]}"
        line_src[cur_line] = r[1].strip()[:90]
        continue
    try:
        s = int(r[4])
    except ValueError:
        continue
    rs = {h[6:]: int(r[i]) for i, h in rs_idx if r[i] not in ("", "-") and int(r[i]) > 0}
    line_tot[cur_line] += s
    line_rs[cur_line].update(rs)
    sass.append((s, r[2], r[3].strip(), cur_line, rs, int(r[7]) if r[7].isdigit() else 0))
tot = sum(line_tot.values())
print(f"total samples {tot}")
allr = collections.Counter()
for c in line_rs.values():
    allr.update(c)
print("all:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in allr.most_common(10)))
for ln, s in line_tot.most_common(n):
    rs = ", ".join(f"{k} {v}" for k, v in line_rs[ln].most_common(4))
    print(f"{100*s/tot:5.1f}% {ln:22s} {line_src.get(ln,'')[:70]} | {rs}")
print("--- top SASS")
for s, addr, ins, ln, rs, ex in sorted(sass, key=lambda x: -x[0])[:n]:
    print(f"{100*s/tot:5.1f}% {ins[:60]:60s} {ln} exec={ex} | " + ", ".join(f"{k} {v}" for k, v in sorted(rs.items(), key=lambda x: -x[1])[:3]))
