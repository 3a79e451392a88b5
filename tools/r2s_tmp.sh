for sc in -1 0 74; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2957$((sc+2)) \
    bench.py --gpus 2 --no-cpu-baseline --e2e-steps 1 --opt shuffle_ctas=$sc > gpurun_out/r2s_sc$sc.json 2> gpurun_out/r2s_sc$sc.err
  echo "[shuffle_ctas=$sc]"; python tools/tools_show_bench.py gpurun_out/r2s_sc$sc.json 2>/dev/null | head -5
done
