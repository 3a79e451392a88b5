#!/bin/bash
# A/B of prebuilt library variants on the bench (run via gpurun).  Variants are built
# here with tools/build_variant.sh NAME "NVCC FLAGS" into build_variants/ (git-ignored,
# shipped with the snapshot); each is swapped in as the package's libgjoin.so in turn.
O=gpurun_out; T=${T:-ab}
cp paper_1904_11201_b200/libgjoin.so /tmp/libgjoin.orig.so
for f in build_variants/libgjoin_*.so; do
  v=$(basename $f .so); v=${v#libgjoin_}
  cp $f paper_1904_11201_b200/libgjoin.so
  timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 --steps 10 ${BENCH_ARGS} > $O/${T}_$v.json 2> $O/${T}_$v.err || tail -3 $O/${T}_$v.err
  echo "[$v]"; python tools/tools_show_bench.py $O/${T}_$v.json 2>/dev/null | head -${LINES_SHOWN:-6}
done
cp /tmp/libgjoin.orig.so paper_1904_11201_b200/libgjoin.so
