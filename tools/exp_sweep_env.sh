#!/bin/bash
# bench configs[1] under several env settings (';'-separated in $ENVS), print step + scatter time
IFS=';' read -ra V <<< "$ENVS"
for e in "${V[@]}"; do
  env $e python bench.py --no-cpu-baseline --e2e-steps 1 --steps 10 ${BENCH_ARGS} > gpurun_out/env.json 2>gpurun_out/env.err || tail -3 gpurun_out/env.err
  python tools/tools_show_bench.py gpurun_out/env.json 2>/dev/null | head -${LINES_SHOWN:-3} | sed "s|^|[$e] |" | sed 's/roofline.*//'
done
