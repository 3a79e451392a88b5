#!/bin/bash
# N-GPU A/B of env settings on a workload (run via gpurun --gpus N): ENVS=';'-separated
N=${N:-2}; WL=${WL:-c2}
IFS=';' read -ra V <<< "$ENVS"
for e in "${V[@]}"; do
  env $e python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N \
    bench.py --gpus $N --workload $WL --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/abd.json 2> gpurun_out/abd.err || tail -5 gpurun_out/abd.err
  python tools/tools_show_bench.py gpurun_out/abd.json 2>/dev/null | head -${LINES_SHOWN:-5} | sed "s|^|[$e] |" | sed 's/roofline.*//'
done
