#!/bin/bash
# A/B of GJ_OPT_SHUFFLE_CTAS (CTAs of the S shuffle scatter that overlaps R's local
# passes) at N GPUs (gpurun --gpus N).  Lines under gpurun_out/${T}_sc<V>.json.
O=gpurun_out; T=${T:-sca}; N=$(nvidia-smi -L | wc -l); P=29600
for V in ${VALS:--1 0 74 148 296}; do
  P=$((P + 1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
    bench.py --gpus $N --workload ${WL:-c2} --no-cpu-baseline --e2e-steps 1 --opt shuffle_ctas=$V \
    > $O/${T}_sc$V.json 2> $O/${T}_sc$V.err
  echo "shuffle_ctas=$V: $(python -c "import json;d=json.load(open('$O/${T}_sc$V.json'));print(round(d['ms_per_step'],3),'ms')" 2>&1 | tail -1)"
done
