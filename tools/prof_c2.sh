#!/bin/bash
# ncu evidence for configs[1] (and the configs[4] shape launch list), current code.
# Usage: R=r01b bash tools/prof_c2.sh   (run via gpurun; plain runs must exit 0 first)
R=${R:-r01}
O=gpurun_out
ARGS="--steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
python bench.py --workload c2 $ARGS > $O/plain_c2.json 2> $O/plain_c2.err || { echo "plain c2 failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches_c2.csv \
    python bench.py --workload c2 $ARGS > $O/ncu_list_c2.log 2>&1 || echo "launch list c2 failed"
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"part_scatter|hj_count_kernel|hj_write_kernel|part_hist" -s 24 -c 8 -o $O/${R}_full_c2 \
    python bench.py --workload c2 $ARGS > $O/ncu_full_c2.log 2>&1 || echo "full c2 failed"
python bench.py --workload c5 --c5-bits 26 $ARGS > $O/plain_c5.json 2> $O/plain_c5.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches_c5.csv \
    python bench.py --workload c5 --c5-bits 26 $ARGS > $O/ncu_list_c5.log 2>&1 || echo "c5 failed"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pf_count|pf_write|bloom_build" \
    -s 3 -c 3 -o $O/${R}_full_c5 python bench.py --workload c5 --c5-bits 26 $ARGS > $O/ncu_full_c5.log 2>&1 || echo "full c5 failed"
ls -la $O | grep $R
