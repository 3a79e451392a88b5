"""PCIe copy rates on the box: pinned H2D / D2H of 1 GiB alone and concurrently (two streams)."""
import time

import torch

n = 1 << 28
h1 = torch.empty(n, dtype=torch.int32).pin_memory()
h2 = torch.empty(n, dtype=torch.int32).pin_memory()
d1 = torch.empty(n, dtype=torch.int32, device="cuda")
d2 = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(f, reps=5):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


gb = n * 4 / 1e9
print(f"H2D alone  {gb / t(lambda: d1.copy_(h1, non_blocking=True)):.1f} GB/s")
print(f"D2H alone  {gb / t(lambda: h2.copy_(d2, non_blocking=True)):.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


print(f"H2D+D2H concurrent: {2 * gb / t(both):.1f} GB/s total")
