"""Aggregate an ncu mixed source page (--print-source cuda,sass) per CUDA line.

  ncu -i rep --page source --csv --print-source cuda,sass > mix.csv
  python tools/ncu_lines.py mix.csv [N]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur_file = cur_line = cur_src = None
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0].strip():
        cur_line, cur_src = (cur_file, int(r[0])), r[1]
        continue
    try:
        ie, sa = float(r[7] or 0), float(r[4] or 0)
    except (ValueError, IndexError):
        continue
    a = agg[cur_line]
    a[0] += ie
    a[1] += sa
    a[2] = cur_src
T = sum(v[0] for v in agg.values())
S = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {T:.4g}")
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f"{v[0] / T * 100:5.1f}% inst {v[1] / S * 100:5.1f}% samp {k[0]}:{k[1]}  {v[2].strip()[:90]}")
