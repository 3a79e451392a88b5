#!/bin/bash
# part_hist CTAs/SM register budget A/B (run via gpurun): C2 x3, C3
for r in 1 2 3; do T=hm$r LINES_SHOWN=3 bash tools/ab_libs.sh; done
T=hmc3 BENCH_ARGS="--workload c3" LINES_SHOWN=1 bash tools/ab_libs.sh
