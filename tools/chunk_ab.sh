#!/bin/bash
# partition chunk size A/B (run via gpurun): parity subset per variant, then C2 twice
O=gpurun_out
cp paper_1904_11201_b200/libgjoin.so /tmp/libgjoin.orig.so
for f in build_variants/libgjoin_*.so; do
  v=$(basename $f .so); v=${v#libgjoin_}
  cp $f paper_1904_11201_b200/libgjoin.so
  timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "equi or partition or shuffle or band or region or prefilter" > $O/chab_pytest_$v.log 2>&1; echo "[$v] pytest rc=$?"; tail -1 $O/chab_pytest_$v.log
done
cp /tmp/libgjoin.orig.so paper_1904_11201_b200/libgjoin.so
T=chab LINES_SHOWN=6 bash tools/ab_libs.sh
T=chab2 LINES_SHOWN=6 bash tools/ab_libs.sh
