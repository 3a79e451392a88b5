#!/bin/bash
# GPU validation pass (run via gpurun): parity suite, smoke, default bench; with >= 2 GPUs
# also the N=2 bench.  Logs under gpurun_out/${TAG}_*.
O=gpurun_out; T=${TAG:-chk}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${T}_smi.txt 2>&1
if [ -n "$PYTEST_K" ]; then KARGS=(-k "$PYTEST_K"); else KARGS=(); fi
timeout ${PYTEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q -x -p no:cacheprovider "${KARGS[@]}" > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/${T}_smoke.log
timeout 600 python bench.py ${BENCH_ARGS} > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"
python tools/tools_show_bench.py $O/${T}_bench.json 2>/dev/null | head -20
N=$(nvidia-smi -L | wc -l)
if [ "$N" -ge 2 ] && [ -z "$NO_DIST" ]; then
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $N --no-cpu-baseline > $O/${T}_bench_n$N.json 2> $O/${T}_bench_n$N.err; echo "bench N=$N rc=$?"
  python tools/tools_show_bench.py $O/${T}_bench_n$N.json 2>/dev/null | head -20
fi
