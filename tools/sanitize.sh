#!/bin/bash
# compute-sanitizer passes over configs[0]-size runs of every kernel family (run via gpurun).
O=gpurun_out; T=${T:-san}
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py ${WHAT:-all} \
    > $O/${T}_$tool.log 2>&1; echo "$tool rc=$?"; tail -4 $O/${T}_$tool.log
done
