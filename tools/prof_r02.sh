#!/bin/bash
# Round-2 profile capture (gpurun, one GPU): plain runs first, then the ncu launch list
# of the same command and one --set full capture of the hot kernels per workload.
#   afterwards, here: python tools/ncu_to_profiles.py r02 c2 gpurun_out/r02_launches_c2.csv gpurun_out/r02_full_c2.ncu-rep
R=${R:-r02}; O=gpurun_out
ARGS="--steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
for W in ${WLS:-c2 c3 c4 c5}; do
  XA=""; [ $W = c5 ] && XA="--c5-bits 26"
  python bench.py --workload $W $ARGS $XA > $O/${R}_plain_$W.json 2> $O/${R}_plain_$W.err || { echo "plain $W failed"; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches_$W.csv \
      python bench.py --workload $W $ARGS $XA > $O/${R}_ncu_list_$W.log 2>&1 || echo "launch list $W failed"
  case $W in
    c2) K="part_scatter|hj_count|hj_write|part_hist|tile_base"; SK=30; CN=7 ;;
    c3) K="part_scatter|hj_count|hj_write"; SK=12; CN=6 ;;
    c4) K="band_|part_scatter"; SK=8; CN=4 ;;
    c5) K="pf_count|pf_write|bloom_build|hj_count"; SK=6; CN=5 ;;
  esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $SK -c $CN \
    -o $O/${R}_full_$W python bench.py --workload $W $ARGS $XA > $O/${R}_ncu_full_$W.log 2>&1 || echo "full $W failed"
done
ls -la $O | grep $R
