#!/bin/bash
# Round profile capture (run on the GPU box via gpurun, one GPU):
#   1. plain bench runs (must exit 0 before any ncu pass),
#   2. the ncu launch list of the same command (gpu__time_duration.sum, clocks uncontrolled),
#   3. one `ncu --set full` capture of each hot kernel.
# Usage: R=r01 bash tools/prof_round.sh
R=${R:-r01}
O=gpurun_out
ARGS="--steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
set -o pipefail
for W in c2 c4; do
  python bench.py --workload $W $ARGS > $O/plain_$W.json 2> $O/plain_$W.err || { echo "plain $W failed"; exit 1; }
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches_$W.csv \
      python bench.py --workload $W $ARGS > $O/ncu_list_$W.log 2>&1 || echo "launch list $W failed"
done
ncu --set full --clock-control none --import-source on -k regex:"part_scatter|hj_count_kernel|hj_write_kernel|part_hist" \
    -s 24 -c 8 -o $O/${R}_full_c2 python bench.py --workload c2 $ARGS > $O/ncu_full_c2.log 2>&1 || echo "full c2 failed"
ncu --set full --clock-control none --import-source on -k regex:"nlj_kernel" \
    -s 2 -c 2 -o $O/${R}_full_c4 python bench.py --workload c4 --c4-s-bits 20 $ARGS > $O/ncu_full_c4.log 2>&1 || echo "full c4 failed"
ls -la $O | tail -20
