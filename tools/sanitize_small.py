"""Small configs[0]-size runs of every kernel family, for compute-sanitizer (memcheck /
racecheck / synccheck) on the GPU box:
    compute-sanitizer --tool memcheck python tools/sanitize_small.py [equi|theta|pf|all]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1904_11201_b200 as gj  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
ctx = gj.Context(0)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
R, S = gen.c1(n=10_000, D=10_000)
tR, tS = dev(R), dev(S)
if what in ("equi", "all"):
    for bits in (-1, 0, 10):
        ctx.set_option("part_bits", bits)
        n = gj.join_count(ctx, tR, tS)
        gj.join_materialize(ctx, tR, tS, n)
        gj.join_materialize(ctx, tR[1:], tS[3:])
    ctx.set_option("part_bits", -1)
    Rp, Sp, _ = gen.pkfk(16, 1 << 16)
    gj.join_materialize(ctx, dev(Rp), dev(Sp))
    gj.join_materialize(ctx, dev(Rp.astype(np.int64)), dev(Sp.astype(np.int64)))
    print("equi ok", flush=True)
if what in ("theta", "all"):
    for op in ("eq", "ne", "lt", "le", "gt", "ge", "band"):
        n = gj.theta_join_count(ctx, tR, tS, op, 3)
        if n < 30_000_000:
            gj.theta_join_materialize(ctx, tR, tS, op, 3, n)
    ctx.set_option("theta_regions", 0)
    gj.theta_join_materialize(ctx, tR, tS, "band", 3)
    print("theta ok", flush=True)
if what in ("pf", "all"):
    R5, S5, _ = gen.c5(1 << 14, 1 << 15, b=14)
    for flags in (1, 3, 7, 8, 12):
        gj.prefilter(ctx, dev(R5), dev(S5), flags)
    pairs = gj.join_materialize(ctx, tR, tS)
    gj.gather_payloads(ctx, pairs, tR, tS)
    print("pf ok", flush=True)
torch.cuda.synchronize()
ctx.close()
print("sanitize_small done")
