#!/bin/bash
# Multi-GPU evidence (run via gpurun --gpus N): NVLink peer-store bandwidth, NCCL a2a,
# the NCCL parity tests, and weak-scaling bench lines.  Logs under gpurun_out/${T}_*.
O=gpurun_out; T=${T:-dist}; N=$(nvidia-smi -L | wc -l)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_nvlink tools/mb_nvlink.cu && /tmp/mb_nvlink > $O/${T}_nvlink.txt 2>&1; cat $O/${T}_nvlink.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 \
  tools/nccl_bench.py > $O/${T}_nccl.txt 2>&1; tail -6 $O/${T}_nccl.txt
if [ -z "$NO_TESTS" ]; then
  timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -p no:cacheprovider > $O/${T}_pytest_dist.log 2>&1; echo "dist pytest rc=$?"; tail -2 $O/${T}_pytest_dist.log
fi
for WL in ${WLS:-c2}; do
  XA=""; [ "$WL" = "c3w" ] && XA="--c3-weak" && W2=c3 || W2=$WL
  timeout 900 python bench.py --workload $W2 $XA --no-cpu-baseline > $O/${T}_${WL}_n1.json 2> $O/${T}_${WL}_n1.err; echo "$WL N=1 rc=$?"
  python tools/tools_show_bench.py $O/${T}_${WL}_n1.json 2>/dev/null | head -3
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29542 \
    bench.py --gpus $N --workload $W2 $XA --no-cpu-baseline > $O/${T}_${WL}_n$N.json 2> $O/${T}_${WL}_n$N.err; echo "$WL N=$N rc=$?"
  python tools/tools_show_bench.py $O/${T}_${WL}_n$N.json 2>/dev/null | head -6
done
