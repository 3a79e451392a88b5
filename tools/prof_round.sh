#!/bin/bash
# Round profile capture (run on the GPU box via gpurun, one GPU):
#   1. plain bench runs (must exit 0 before any ncu pass),
#   2. the ncu launch list of the same command (gpu__time_duration.sum, clocks uncontrolled),
#   3. one `ncu --set full` capture of each hot kernel.
# Usage: R=r01 bash tools/prof_round.sh   then, here:
#   python tools/ncu_to_profiles.py r01 c2 gpurun_out/r01_launches_c2.csv gpurun_out/r01_full_c2.ncu-rep  (c4, c5 alike)
R=${R:-r01}
O=gpurun_out
ARGS="--steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
set -o pipefail
for W in c2 c4 c5; do
  XA=""; [ $W = c5 ] && XA="--c5-bits 26"
  python bench.py --workload $W $ARGS $XA > $O/plain_$W.json 2> $O/plain_$W.err || { echo "plain $W failed"; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches_$W.csv \
      python bench.py --workload $W $ARGS $XA > $O/ncu_list_$W.log 2>&1 || echo "launch list $W failed"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"part_scatter|hj_count|hj_write|part_hist|tile_base" \
    -s 30 -c 6 -o $O/${R}_full_c2 python bench.py --workload c2 $ARGS > $O/ncu_full_c2.log 2>&1 || echo "full c2 failed"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"nlj_kernel|part_scatter" \
    -s 8 -c 4 -o $O/${R}_full_c4 python bench.py --workload c4 $ARGS > $O/ncu_full_c4.log 2>&1 || echo "full c4 failed"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pf_count|pf_write|bloom_build" \
    -s 6 -c 4 -o $O/${R}_full_c5 python bench.py --workload c5 --c5-bits 26 $ARGS > $O/ncu_full_c5.log 2>&1 || echo "full c5 failed"
ls -la $O | grep $R
