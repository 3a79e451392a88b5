TAG=r2r NO_DIST=1 PYTEST_K="theta or golden or band or region" BENCH_ARGS="--workload c4" bash tools/gpu_check.sh
T=r2r_hj KREGEX="hj_count|hj_write" SKIP=3 COUNT=2 bash tools/prof_kernels.sh
