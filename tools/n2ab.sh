#!/bin/bash
O=gpurun_out; T=${T:-n2ab}; N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -p no:cacheprovider > $O/${T}_pytest_dist.log 2>&1; echo "dist pytest rc=$?"; tail -2 $O/${T}_pytest_dist.log
cp paper_1904_11201_b200/libgjoin.so /tmp/libgjoin.orig.so
for rep in 1 2; do
for v in ovl noovl; do
  cp build_variants/libgjoin_$v.so paper_1904_11201_b200/libgjoin.so
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$rep \
    bench.py --gpus $N --no-cpu-baseline --e2e-steps 1 > $O/${T}_${v}_$rep.json 2> $O/${T}_${v}_$rep.err; echo "[$v $rep] rc=$?"
  python tools/tools_show_bench.py $O/${T}_${v}_$rep.json 2>/dev/null | head -4
done; done
cp /tmp/libgjoin.orig.so paper_1904_11201_b200/libgjoin.so
