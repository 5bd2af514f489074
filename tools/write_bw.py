"""Pure-write HBM bandwidth on this GPU (context for the write-dominated window kernel).

fill_ / zero_ of a 3.69 GB fp32 tensor (the size of 1000 C3 surfaces), best of 10, CUDA events.
"""
import json

import torch

n = 1000 * 1280 * 720
x = torch.empty(n, dtype=torch.float32, device="cuda")
res = {}
for name, fn in (("fill_", lambda: x.fill_(1.0)), ("zero_", lambda: x.zero_())):
    for _ in range(3):
        fn()
    best = 1e9
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    res[name] = {"ms": best, "gbs": n * 4 / best / 1e6}
print(json.dumps(res))
