#!/bin/bash
# microbenchmarks on the GPU box (run via gpurun): INT peak + smem table ops
O=gpurun_out; T=${T:-mb}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_ops tools/mb_ops.cu && /tmp/mb_ops > $O/${T}_mb_ops.txt 2>&1
cat $O/${T}_mb_ops.txt
