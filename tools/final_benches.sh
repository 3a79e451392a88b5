#!/bin/bash
# Round-end bench lines on one GPU (gpurun): every workload with its CPU baseline, plus
# the reference arm of the default workload.  Outputs gpurun_out/${T}_*.json
O=gpurun_out; T=${T:-fin}
for W in ${WLS:-c2 c3 c4 c5 c1}; do
  timeout 900 python bench.py --workload $W > $O/${T}_$W.json 2> $O/${T}_$W.err; echo "$W rc=$?"
  python tools/tools_show_bench.py $O/${T}_$W.json 2>/dev/null | head -4
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/${T}_ref.json 2> $O/${T}_ref.err; echo "ref rc=$?"; cat $O/${T}_ref.json | head -c 600; echo
