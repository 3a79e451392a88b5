R=r01; O=gpurun_out; ARGS="--steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
python bench.py --workload c5 --c5-bits 26 $ARGS > $O/plain_c5.json 2> $O/plain_c5.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches_c5.csv python bench.py --workload c5 --c5-bits 26 $ARGS > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pf_count|pf_write|bloom_build" -s 6 -c 4 -o $O/${R}_full_c5 python bench.py --workload c5 --c5-bits 26 $ARGS > /dev/null 2>&1
ls -la $O | grep r01
