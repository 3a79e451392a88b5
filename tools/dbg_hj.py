"""Debug helper (GPU): hj_count time on C2 keys vs the keys one rank receives at N=2
(perm_28 domain, top khash bit 0), same partition sizes.  python tools/dbg_hj.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import gen.device as gd  # noqa: E402
import paper_1904_11201_b200 as gj  # noqa: E402

C1 = 0x9E3779B97F4A7C15 - (1 << 64)  # as int64


def top_bit_zero(k):
    p = (k.to(torch.int64) & 0xFFFFFFFF) * C1  # wraps mod 2^64
    return p >= 0


def run(name, R, S, **opts):
    ctx = gj.Context(0, torch.cuda.current_stream(), **opts)
    Rr, Sr = gj.Rel(R), gj.Rel(S)
    for _ in range(2):
        n = gj.join_count(ctx, Rr, Sr)
    ctx.set_option("profile", 1)
    ctx.reset_stats()
    for _ in range(5):
        n = gj.join_count(ctx, Rr, Sr)
    kt = ctx.kernel_times()
    print(name, "n", n, {k: round(v[0] / v[1], 4) for k, v in kt.items() if k in ("hj_count", "part_scatter", "part_hist")},
          flush=True)
    ctx.close()


seed = gen.BASE_SEED
n = 1 << 27
run("c2 B=auto", gd.perm_range(n, 27, seed), gd.pkfk_S(n, 27, seed))
R2 = gd.perm_range(2 * n, 28, seed)
S2 = gd.pkfk_S(2 * n, 28, seed)
R2 = R2[top_bit_zero(R2)].contiguous()
S2 = S2[top_bit_zero(S2)].contiguous()
print("rank0-like sizes", R2.numel(), S2.numel())
run("n2-like B=18", R2, S2, part_bits=18)
run("c2 B=17 explicit", gd.perm_range(n, 27, seed), gd.pkfk_S(n, 27, seed), part_bits=17)
R3 = gd.perm_range(n, 27, seed)
S3 = gd.pkfk_S(n, 27, seed)
run("c2 B=18", R3, S3, part_bits=18)
