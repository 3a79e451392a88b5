#!/bin/bash
# ncu capture of the main C2 kernels (run via gpurun); the plain run must exit 0 first
ARGS="--steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS}"
python bench.py $ARGS > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-part_scatter|hj_kernel|part_hist}" -s ${SKIP:-30} -c ${COUNT:-8} -o gpurun_out/${OUT:-prof} python bench.py $ARGS > gpurun_out/prof_ncu.log 2>&1
tail -2 gpurun_out/prof_ncu.log
