"""Opcode mix of one kernel from `ncu --page source --csv` (SASS view): % of executed
instructions and % of stall samples per opcode.  Usage: tools_ncu_ops.py dump.csv"""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
c, s = Counter(), Counter()
for r in rows:
    if "Instructions Executed" in r:
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr) // 2:
        continue
    try:
        ie = float(r[hdr["Instructions Executed"]] or 0)
        sp = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    toks = r[hdr["Source"]].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    c[op] += ie
    s[op] += sp
tot, ts = sum(c.values()), sum(s.values())
print(f"total executed {tot:.3g}  stall samples {ts:.3g}")
for k, v in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{k:28s} {v/tot*100:5.1f}% inst  {s[k]/ts*100:5.1f}% samples")
