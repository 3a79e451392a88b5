#!/bin/bash
# programmatic dependent launch A/B (run via gpurun): full GPU suite on the built lib (PDL on), then C2 x3, C3, C4, C5
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pdl_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pdl_pytest.log
for r in 1 2 3; do T=pdl$r LINES_SHOWN=1 bash tools/ab_libs.sh; done
for W in c3 c4 c5; do T=pdl$W BENCH_ARGS="--workload $W" LINES_SHOWN=1 bash tools/ab_libs.sh; done
