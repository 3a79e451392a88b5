#!/bin/bash
# join_count_materialize (one C-ABI call) vs join_count + join_materialize (run via gpurun)
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "count_materialize or c2_full or slot_const" > $O/fu_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/fu_pytest.log
for rep in 1 2; do
  for W in c2 c5; do
    timeout 600 python bench.py --workload $W --no-cpu-baseline --e2e-steps 1 > $O/fu_${W}_one_$rep.json 2> $O/fu_${W}_one_$rep.err; echo "[$W one-call $rep] rc=$?"
    python tools/tools_show_bench.py $O/fu_${W}_one_$rep.json 2>/dev/null | head -1 | cut -c1-60
    timeout 600 python bench.py --workload $W --no-cpu-baseline --e2e-steps 1 --two-call-step > $O/fu_${W}_two_$rep.json 2> $O/fu_${W}_two_$rep.err; echo "[$W two-call $rep] rc=$?"
    python tools/tools_show_bench.py $O/fu_${W}_two_$rep.json 2>/dev/null | head -1 | cut -c1-60
  done
done
