"""Aggregate an ncu source-page CSV (SASS view: Address, samples, instructions)
by CUDA source line, using `nvdisasm -g` line info of the same build
(measurement tool).

    python tools/sass_lines.py all.sass <mangled-kernel-substring> page.csv [top]
"""
import collections
import csv
import re
import sys

sass, kern, page = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
addr2line = {}
inside = False
cur = None
for ln in open(sass):
    if ln.startswith(".text."):
        inside = kern in ln
        continue
    if not inside:
        continue
    m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        addr2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(page)))
h = rows[1]
ia, isamp, iinst = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
agg = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter()])
tot_s = tot_i = 0.0
base = None
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
    except ValueError:
        continue
    if base is None:
        base = a
    a -= base  # (the page gives load addresses; nvdisasm offsets from the function start)
    key = addr2line.get(a, ("?", 0))
    s = float(r[isamp] or 0)
    n = float(r[iinst] or 0)
    agg[key][0] += s
    agg[key][1] += n
    for i in stall_cols:
        v = float(r[i] or 0)
        if v:
            agg[key][2][h[i][6:]] += v
    tot_s += s
    tot_i += n
print(f"total samples {tot_s:.0f}, warp instructions {tot_i:.4g}")
for key, (s, n, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    tops = ", ".join(f"{k} {v / max(s, 1):.2f}" for k, v in st.most_common(3))
    print(f"{key[0]}:{key[1]:5d}  samples {100 * s / tot_s:5.1f}%  inst {100 * n / tot_i:5.1f}%  [{tops}]")
