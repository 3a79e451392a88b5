for h in 0 1 2 3; do
  GJ_L2HINT=$h GJ_SCATTER_V=4 python bench.py --no-cpu-baseline --e2e-steps 1 --steps 10 > gpurun_out/h$h.json 2>gpurun_out/h$h.err
  echo "[hint $h]"; python tools/tools_show_bench.py gpurun_out/h$h.json 2>/dev/null | sed -n 2p
done
for h in 1 3; do GJ_L2HINT=$h VARIANTS=4 bash tools/ab_ncu.sh | sed "s/^/h$h /"; done
