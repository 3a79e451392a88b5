#!/bin/bash
# NEXT row f4: the paper's alpha study (PAPER.md:330-336, :358-363 -- reducer count vs
# time) on configs[1]: partition bits B (2^B partitions = "reducers") x work-unit
# capacity.  Run via gpurun; prints one line per setting.
for cfg in "part_bits=14 build_chunk=4096 probe_chunk=4096" "part_bits=15 build_chunk=4096 probe_chunk=4096" \
           "part_bits=16 build_chunk=4096 probe_chunk=4096" "part_bits=17 build_chunk=2048 probe_chunk=2048" \
           "part_bits=18 build_chunk=1024 probe_chunk=1024" "part_bits=16 build_chunk=4096 probe_chunk=1024"; do
  args=""; for o in $cfg; do args="$args --opt $o"; done
  python bench.py --no-cpu-baseline --e2e-steps 1 --steps 10 $args > gpurun_out/gran.json 2>gpurun_out/gran.err || { tail -3 gpurun_out/gran.err; continue; }
  python - "$cfg" << 'PY'
import json, sys
d = json.load(open("gpurun_out/gran.json"))
k = d["kernels"]
f = lambda t: k.get(t, {}).get("ms_per_launch", 0) * k.get(t, {}).get("launches_per_step", 0)
print(f"| {sys.argv[1]} | {d['ms_per_step']:.3f} | {d['value']/1e9:.1f} | {f('part_hist')+f('tile_base'):.3f} | "
      f"{f('part_scatter'):.3f} | {f('hj_count'):.3f} | {f('hj_write')+f('hj_write_multi'):.3f} |")
PY
done
