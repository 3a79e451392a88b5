python tools/dbg_hj.py both > gpurun_out/r2p_dbg.txt 2>&1; cat gpurun_out/r2p_dbg.txt
TAG=r2p NO_DIST=1 PYTEST_K="equi or golden or join or gather or stats or unaligned or host or launch or c5 or alloc" bash tools/gpu_check.sh
