"""Attribute ncu SASS-level stall samples / executed instructions to CUDA source lines.

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX SOURCE.cu [N]

Compiles SOURCE.cu to a cubin with -lineinfo, maps every SASS offset of the
kernel to its source line with nvdisasm, and joins that with the per-instruction
metrics of the first matching launch in the report (matched by offset from the
function start).  Prints the top-N source lines.
"""
import csv
import io
import os
import re
import subprocess
import sys
from collections import defaultdict

rep, kre, src = sys.argv[1], sys.argv[2], sys.argv[3]
topn = int(sys.argv[4]) if len(sys.argv) > 4 else 30
which = int(sys.argv[5]) if len(sys.argv) > 5 else 0  # index of the matching launch in the report
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cubin = "/tmp/_lines.cubin"
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                       "-std=c++17", "--expt-relaxed-constexpr", "-I", os.path.join(root, "include"), "-I",
                       os.path.dirname(os.path.abspath(src)), "-cubin", "-o", cubin, src])
dis = subprocess.run(["/usr/local/cuda/bin/nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# split per function
funcs = {}
cur = None
line = None
for l in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        cur = m.group(1)
        funcs[cur] = {}
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = int(m.group(2))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m and cur:
        funcs[cur][int(m.group(1), 16)] = (line, m.group(2).strip())

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
kname = None
hdr = None
recs = []
for r in rows:
    if r and r[0] == "Kernel Name":
        which -= 1
        if which < -1:
            break
        kname = r[1]
        recs = []
        continue
    if "Address" in r and "Source" in r:
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr and which == -1 and len(r) >= len(hdr) // 2:
        try:
            recs.append((int(r[hdr["Address"]], 16), r[hdr["Source"]].strip(),
                         float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0),
                         float(r[hdr["Instructions Executed"]] or 0)))
        except ValueError:
            pass
base = min(a for a, *_ in recs)
# pick the cubin function whose instruction sequence matches best
best, score = None, -1
for fn, ins in funcs.items():
    s = sum(1 for a, sass, *_ in recs if (a - base) in ins and ins[a - base][1].split()[0] in sass)
    if s > score:
        best, score = fn, s
ins = funcs[best]
agg = defaultdict(lambda: [0.0, 0.0])
ts = sum(r[2] for r in recs) or 1
te = sum(r[3] for r in recs) or 1
for a, sass, s, e in recs:
    ln = ins.get(a - base, (None, ""))[0]
    agg[ln][0] += s
    agg[ln][1] += e
srclines = open(src).read().splitlines()
print(f"kernel {kname[:80]}\nmatched {best} ({score}/{len(recs)} instructions)")
for ln, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:topn]:
    text = srclines[ln - 1].strip()[:90] if ln and ln <= len(srclines) else "?"
    print(f"{s/ts*100:5.1f}% stall {e/te*100:5.1f}% inst  L{ln}: {text}")
