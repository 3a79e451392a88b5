#!/bin/bash
# second-stream priority A/B (run via gpurun): C2 x3, C3, C5
for r in 1 2 3; do T=prio$r LINES_SHOWN=1 bash tools/ab_libs.sh; done
T=prioc3 BENCH_ARGS="--workload c3" LINES_SHOWN=1 bash tools/ab_libs.sh
T=prioc5 BENCH_ARGS="--workload c5" LINES_SHOWN=1 bash tools/ab_libs.sh
