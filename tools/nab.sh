#!/bin/bash
# multi-GPU A/B of prebuilt library variants (run via gpurun --gpus N): C2 weak bench per variant, twice
O=gpurun_out; T=${T:-nab}; N=$(nvidia-smi -L | wc -l)
cp paper_1904_11201_b200/libgjoin.so /tmp/libgjoin.orig.so
for rep in 1 2; do
for f in build_variants/libgjoin_*.so; do
  v=$(basename $f .so); v=${v#libgjoin_}
  cp $f paper_1904_11201_b200/libgjoin.so
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$rep \
    bench.py --gpus $N --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS} > $O/${T}_${v}_$rep.json 2> $O/${T}_${v}_$rep.err; echo "[$v $rep] rc=$?"
  python tools/tools_show_bench.py $O/${T}_${v}_$rep.json 2>/dev/null | head -${LINES_SHOWN:-1} | cut -c1-60
done; done
cp /tmp/libgjoin.orig.so paper_1904_11201_b200/libgjoin.so
