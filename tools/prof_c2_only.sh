#!/bin/bash
# configs[1] ncu evidence only (launch list + one --set full capture of the hot kernels).
# Usage: R=r01 bash tools/prof_c2_only.sh   (run via gpurun; the plain run must exit 0 first)
R=${R:-r01}
O=gpurun_out
ARGS="--steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
python bench.py --workload c2 $ARGS > $O/plain_c2.json 2> $O/plain_c2.err || { echo "plain c2 failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches_c2.csv \
    python bench.py --workload c2 $ARGS > $O/ncu_list_c2.log 2>&1 || echo "launch list c2 failed"
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"part_scatter|hj_count_kernel|hj_write_fast|part_hist" -s 24 -c 8 -o $O/${R}_full_c2 \
    python bench.py --workload c2 $ARGS > $O/ncu_full_c2.log 2>&1 || echo "full c2 failed"
ls -la $O | grep $R
