"""Summarise an `ncu --page source --csv` dump: top SASS lines by stall samples and stall totals."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ci = {h: i for i, h in enumerate(hdr)}
samp = ci["Warp Stall Sampling (All Samples)"]
tot = 0
stalls = {}
for r in data:
    try:
        s = float(r[samp] or 0)
    except ValueError:
        continue
    tot += s
    for h, i in ci.items():
        if i >= len(r): continue
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                stalls[h] = stalls.get(h, 0) + float(r[i] or 0)
            except ValueError:
                pass
print("total samples", tot)
for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {k:28s} {v/tot*100:5.1f}%")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
top = sorted(data, key=lambda r: -float(r[samp] or 0) if r[samp].replace('.', '', 1).isdigit() else 0)[:n]
for r in top:
    print(f"{float(r[samp] or 0)/tot*100:5.1f}%  {r[ci['Address']]:>6s}  {r[ci['Source']][:90]}")
