python tools/dbg_hj.py both > gpurun_out/r2n_dbg.txt 2>&1; cat gpurun_out/r2n_dbg.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hj_count -s 3 -c 1 -o gpurun_out/r2n_n2 python tools/dbg_hj.py n2 > gpurun_out/r2n_ncu.log 2>&1; echo ncu rc=$?
python tools/tools_ncu_summary.py gpurun_out/r2n_n2.ncu-rep 2>&1 | head -25
T=r2n LINES_SHOWN=5 bash tools/ab_libs.sh
