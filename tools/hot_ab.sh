#!/bin/bash
# skewed-tile ranking A/B (run via gpurun): parity subset on the built lib, then C2 / C3 / C4-skew per variant
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/hot_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/hot_pytest.log
T=hotc2 LINES_SHOWN=3 bash tools/ab_libs.sh
T=hotc3 BENCH_ARGS="--workload c3" LINES_SHOWN=3 bash tools/ab_libs.sh
T=hotc2b LINES_SHOWN=1 bash tools/ab_libs.sh
T=hotc3b BENCH_ARGS="--workload c3" LINES_SHOWN=1 bash tools/ab_libs.sh
