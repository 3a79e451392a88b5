#!/bin/bash
# A/B of prebuilt library variants (build_variants/libgjoin_*.so, git-ignored) on the
# bench (run via gpurun): each is swapped in as the package's libgjoin.so in turn.
cp paper_1904_11201_b200/libgjoin.so /tmp/libgjoin.orig.so
for f in build_variants/libgjoin_*.so; do
  cp "$f" paper_1904_11201_b200/libgjoin.so
  python bench.py --no-cpu-baseline --e2e-steps 1 --steps 10 ${BENCH_ARGS} > gpurun_out/abl.json 2> gpurun_out/abl.err || tail -3 gpurun_out/abl.err
  python tools/tools_show_bench.py gpurun_out/abl.json 2>/dev/null | head -${LINES_SHOWN:-6} | sed "s|^|[$(basename $f)] |" | sed 's/roofline.*//'
done
cp /tmp/libgjoin.orig.so paper_1904_11201_b200/libgjoin.so
