#!/bin/bash
# Device timeline of one profiled step (GJ_TRACE=3) at N = #GPUs (run via gpurun): C2 by default
O=gpurun_out; T=${T:-tl}; N=$(nvidia-smi -L | wc -l)
if [ "$N" -ge 2 ]; then
  GJ_TRACE=3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29551 \
    bench.py --gpus $N --no-cpu-baseline --e2e-steps 1 --steps 3 ${BENCH_ARGS} > $O/${T}_n$N.json 2> $O/${T}_n$N.err; echo "rc=$?"
else
  GJ_TRACE=3 timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 --steps 3 ${BENCH_ARGS} > $O/${T}_n1.json 2> $O/${T}_n1.err; echo "rc=$?"
fi
grep -c "gj tl" $O/${T}_n$N.err
