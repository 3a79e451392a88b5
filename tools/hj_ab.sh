#!/bin/bash
# hash-table slots-per-row A/B on C2 dense and sparse keys (run via gpurun)
T=hja LINES_SHOWN=5 bash tools/ab_libs.sh
T=hjs BENCH_ARGS="--c2-sparse" LINES_SHOWN=5 bash tools/ab_libs.sh
T=hja2 LINES_SHOWN=5 bash tools/ab_libs.sh
