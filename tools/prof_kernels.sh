#!/bin/bash
# ncu --set full capture of selected kernels of one bench workload (run via gpurun, 1 GPU;
# the plain run must exit 0 first).  KREGEX = kernel-name regex, WL = workload, T = tag.
O=gpurun_out; T=${T:-prof}; WL=${WL:-c2}
ARGS="--workload $WL --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline ${BENCH_ARGS}"
python bench.py $ARGS > $O/${T}_plain.json 2> $O/${T}_plain.err || { echo "plain run failed"; tail -5 $O/${T}_plain.err; exit 1; }
python tools/tools_show_bench.py $O/${T}_plain.json | head -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-hj_count|hj_write}" \
  -s ${SKIP:-6} -c ${COUNT:-2} -o $O/${T} python bench.py $ARGS > $O/${T}_ncu.log 2>&1; echo "ncu rc=$?"
python tools/tools_ncu_summary.py $O/${T}.ncu-rep > $O/${T}_summary.txt 2>&1; cat $O/${T}_summary.txt | head -80
