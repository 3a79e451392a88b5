#!/bin/bash
# A/B of GJ_OPT_SHUFFLE_BITS (local radix bits folded into the NVLink shuffle) at N
# GPUs (gpurun --gpus N).  Lines under gpurun_out/${T}_sb<V>.json.
O=gpurun_out; T=${T:-sba}; N=$(nvidia-smi -L | wc -l); P=29700
for V in ${VALS:-0 3 5 7}; do
  P=$((P + 1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
    bench.py --gpus $N --workload ${WL:-c2} --no-cpu-baseline --e2e-steps 1 --opt shuffle_bits=$V \
    > $O/${T}_sb$V.json 2> $O/${T}_sb$V.err
  echo "shuffle_bits=$V: $(python -c "
import json;d=json.load(open('$O/${T}_sb$V.json'));k=d['kernels']
print(round(d['ms_per_step'],3),'ms', {t:(round(v['ms_per_launch'],3),v['launches_per_step']) for t,v in k.items() if t in ('shuffle_scatter','part_scatter','part_hist','hj_count')})" 2>&1 | tail -1)"
done
