"""Aggregate an ncu source page (SASS) by opcode and stall reason.

  ncu -i rep --page source --csv --print-source sass > src.csv
  python tools/ncu_stalls.py src.csv [N]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
iS = hdr.index("Source")
iE = hdr.index("Instructions Executed")
cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
by_op = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for r in data:
    src = r[iS].strip().split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") and len(src) > 1 else src[0]
    op = op.split(".")[0]
    for i, h in cols:
        v = float(r[i] or 0)
        by_op[op][h[6:]] += v
        tot[h[6:]] += v
    by_op[op]["_exec"] += float(r[iE] or 0)
T = sum(v for k, v in tot.items())
print("stall share:", {k: round(v / T, 3) for k, v in tot.most_common(8)})
N = int(sys.argv[2]) if len(sys.argv) > 2 else 15
for op, c in sorted(by_op.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "_exec"))[:N]:
    s = sum(v for k, v in c.items() if k != "_exec")
    top = ", ".join(f"{k}={v / T:.3f}" for k, v in c.most_common(5) if k != "_exec")
    print(f"{op:10s} {s / T:6.3f}  exec={int(c['_exec']):>9}  {top}")
