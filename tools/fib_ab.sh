#!/bin/bash
# Fibonacci-slot A/B (run via gpurun): full GPU parity suite on the built lib, then C2 / C3 / C2-sparse per variant
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/fib_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/fib_pytest.log
T=fibc2 LINES_SHOWN=5 bash tools/ab_libs.sh
T=fibc3 BENCH_ARGS="--workload c3" LINES_SHOWN=5 bash tools/ab_libs.sh
T=fibsp BENCH_ARGS="--c2-sparse" LINES_SHOWN=5 bash tools/ab_libs.sh
