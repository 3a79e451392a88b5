#!/bin/bash
# 4-GPU round evidence (gpurun --gpus 4): full GPU parity suite (incl. the world-2/4 NCCL
# tests), configs[4] at full size with the O8 check, NVLink/NCCL at 4 GPUs, weak-scaling lines.
O=gpurun_out; T=${T:-r2n4}
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/${T}_pytest.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 \
  tools/c5_full_dist.py --bits 31 --out $O/${T}_c5_full.json > $O/${T}_c5_full.log 2>&1; echo "c5 full rc=$?"; tail -2 $O/${T}_c5_full.log
NO_TESTS=1 WLS="c2 c3w" T=$T bash tools/dist_check.sh
