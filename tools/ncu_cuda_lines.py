"""Per-CUDA-source-line instruction and stall-sample shares of one kernel, from
`ncu -i rep --page source --csv --print-source cuda,sass -k regex:NAME` (the per-line
rows carry the aggregated metrics).  Usage: ncu_cuda_lines.py dump.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
path, hdr, width, lines = None, None, 0, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = {h: i for i, h in reversed(list(enumerate(r)))}  # first of a duplicated name
        width = len(r)
    elif hdr and len(r) == width and r[0] and r[2] == "-":  # a source line (SASS rows carry an address)
        lines.append((path, r))
ie, sm = hdr["Instructions Executed"], hdr["Warp Stall Sampling (All Samples)"]
f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
tot = sum(f(r[ie]) for _, r in lines)
ts = sum(f(r[sm]) for _, r in lines)
print(f"{tot:.4g} warp instructions, {ts:.4g} stall samples")
for p, r in sorted(lines, key=lambda x: -f(x[1][ie]))[:top]:
    print(f"{f(r[ie]) / tot * 100:5.1f}% st={f(r[sm]) / ts * 100:4.1f}% {p}:{r[0]} {r[1].strip()[:80]}")
