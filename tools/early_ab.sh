#!/bin/bash
# hash-count early probe-vector load A/B (run via gpurun): equi parity subset with e1, then C2 x3, C3, sparse
O=gpurun_out
cp paper_1904_11201_b200/libgjoin.so /tmp/libgjoin.orig.so; cp build_variants/libgjoin_e1.so paper_1904_11201_b200/libgjoin.so
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "equi or join" > $O/early_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/early_pytest.log
cp /tmp/libgjoin.orig.so paper_1904_11201_b200/libgjoin.so
for r in 1 2 3; do T=ea$r LINES_SHOWN=5 bash tools/ab_libs.sh; done
T=eac3 BENCH_ARGS="--workload c3" LINES_SHOWN=5 bash tools/ab_libs.sh
T=easp BENCH_ARGS="--c2-sparse" LINES_SHOWN=5 bash tools/ab_libs.sh
