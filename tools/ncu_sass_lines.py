"""Per-SASS-line executed-instruction and stall-sample shares of one kernel from
`ncu -i rep --page source --csv --print-source sass -k regex:NAME` (first launch only).
Usage: ncu_sass_lines.py dump.csv [min_pct]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 0.25
hdr, data = None, []
for r in rows:
    if "Instructions Executed" in r:
        if hdr is not None:
            break  # second launch: stop
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is not None and len(r) >= len(hdr) - 2:
        data.append(r)
ie, src, th, sm = (hdr[k] for k in ("Instructions Executed", "Source", "Avg. Threads Executed",
                                   "Warp Stall Sampling (All Samples)"))
f = lambda x: float(x or 0)  # noqa: E731
tot, ts = sum(f(r[ie]) for r in data), sum(f(r[sm]) for r in data)
print(f"{len(data)} SASS lines, {tot:.4g} warp instructions, {ts:.4g} stall samples")
for r in data:
    v = f(r[ie])
    if v / tot * 100 >= mn or f(r[sm]) / ts * 100 >= mn:
        print(f"{v / tot * 100:5.2f}% st={f(r[sm]) / ts * 100:4.1f}% thr={f(r[th]):4.1f} {r[src].strip()[:70]}")
