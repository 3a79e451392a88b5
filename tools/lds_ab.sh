#!/bin/bash
# scatter load/store ordering A/B (run via gpurun): partition parity subset per variant, then C2 x3 and C3
O=gpurun_out
cp paper_1904_11201_b200/libgjoin.so /tmp/libgjoin.orig.so
for f in build_variants/libgjoin_*.so; do
  v=$(basename $f .so); v=${v#libgjoin_}
  cp $f paper_1904_11201_b200/libgjoin.so
  timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "equi or shuffle or band or region" > $O/lds_pytest_$v.log 2>&1; echo "[$v] pytest rc=$?"; tail -1 $O/lds_pytest_$v.log
done
cp /tmp/libgjoin.orig.so paper_1904_11201_b200/libgjoin.so
for r in 1 2 3; do T=lds$r LINES_SHOWN=2 bash tools/ab_libs.sh; done
T=lds3c BENCH_ARGS="--workload c3" LINES_SHOWN=1 bash tools/ab_libs.sh
