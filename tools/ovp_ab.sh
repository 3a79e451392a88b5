O=gpurun_out
for rep in 1 2; do for W in c3 c5; do for o in 1 0; do
timeout 600 python bench.py --workload $W --no-cpu-baseline --e2e-steps 1 --opt overlap_partitions=$o > $O/ovp_${W}_${o}_$rep.json 2>$O/ovp_${W}_${o}_$rep.err; echo "[$W ovp=$o $rep] rc=$?"
python tools/tools_show_bench.py $O/ovp_${W}_${o}_$rep.json 2>/dev/null | head -1 | cut -c1-60
done; done; done
