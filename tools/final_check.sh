#!/bin/bash
# Round-end validation on the GPU box: full GPU parity suite, smoke(), default bench, per-workload benches.
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/final_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/final_smoke.log
timeout 600 python bench.py > $O/final_bench.json 2> $O/final_bench.err; echo "bench rc=$?"; cat $O/final_bench.json
for W in c4 c5; do timeout 600 python bench.py --workload $W --no-cpu-baseline > $O/final_bench_$W.json 2> $O/final_bench_$W.err; echo "$W rc=$?"; done
