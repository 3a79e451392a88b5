#!/bin/bash
# A/B of scatter variants on configs[1] (run via gpurun): per-kernel times per variant
for v in ${VARIANTS:-2 4}; do
  GJ_SCATTER_V=$v python bench.py --no-cpu-baseline --e2e-steps 1 --steps 10 ${BENCH_ARGS} > gpurun_out/ab_v$v.json 2>gpurun_out/ab_v$v.err || tail -5 gpurun_out/ab_v$v.err
  echo "[v$v]"; python tools/tools_show_bench.py gpurun_out/ab_v$v.json 2>/dev/null | head -6
done
