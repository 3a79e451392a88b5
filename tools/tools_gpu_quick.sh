#!/bin/bash
# quick GPU iteration: equi/golden parity tests + C2 bench (used via gpurun)
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider --timeout 500 -k "${TESTS:-equi or golden}" > gpurun_out/pytest_quick.log 2>&1
tail -3 gpurun_out/pytest_quick.log
python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -3 gpurun_out/bench_quick.err
