import json, sys
d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else '/root/repo/gpurun_out/bench_quick.json'))
print(f"{d['value']/1e9:.2f} G input tuples/s  {d['ms_per_step']:.3f} ms/step  roofline {d['roofline']}")
for k, v in sorted(d['kernels'].items(), key=lambda kv: -kv[1]['share']):
    print(f"  {k:14s} {v['ms_per_launch']:.4f} ms x{v['launches_per_step']:.0f}  share {v['share']:.3f}  {v.get('achieved_gbs', 0):.0f} GB/s")
