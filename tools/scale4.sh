#!/bin/bash
# N-GPU weak-scaling bench lines for c2, c4, c5 (run via gpurun --gpus N)
N=${N:-4}
for wl in c2 c4 c5; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N \
    bench.py --gpus $N --workload $wl --steps 5 --warmup 3 --e2e-steps 2 > gpurun_out/b${N}_$wl.json 2> gpurun_out/b${N}_$wl.err
  echo "[$wl N=$N]"; python tools/tools_show_bench.py gpurun_out/b${N}_$wl.json 2>/dev/null | head -3
done
python bench.py --workload c5 --steps 5 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/b1_c5.json 2> gpurun_out/b1_c5.err
echo "[c5 N=1]"; python tools/tools_show_bench.py gpurun_out/b1_c5.json 2>/dev/null | head -3
