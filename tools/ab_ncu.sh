#!/bin/bash
# Per-launch time + DRAM bytes of the scatter launches per variant (ncu, cold per launch).
# Run via gpurun.  KREGEX selects kernels (default part_scatter).
for v in ${VARIANTS:-2 4}; do
  GJ_SCATTER_V=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:"${KREGEX:-part_scatter}" -s ${SKIP:-4} -c ${COUNT:-4} --csv \
    python bench.py --workload ${WL:-c2} --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline 2>/dev/null \
    | grep -E '^"[0-9]' | awk -F'","' -v v=$v '{printf "v%s %-40s %-28s %s\n", v, substr($5,1,40), $(NF-2), $NF}'
done
