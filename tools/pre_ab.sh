#!/bin/bash
# scatter column-prefix load ordering A/B under PDL (run via gpurun): C2 x4
for r in 1 2 3 4; do T=pre$r LINES_SHOWN=1 bash tools/ab_libs.sh; done
