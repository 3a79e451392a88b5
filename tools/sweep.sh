#!/bin/bash
# run bench variants (args separated by ';' in $SWEEP) and print step times
IFS=';' read -ra V <<< "$SWEEP"
for v in "${V[@]}"; do
  python bench.py --no-cpu-baseline --e2e-steps 1 --steps 10 $v > gpurun_out/sweep.json 2>/dev/null
  python tools/tools_show_bench.py gpurun_out/sweep.json | head -6 | sed "s|^|[$v] |"
done
