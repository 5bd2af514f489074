"""Surfaces/s at C3 geometry for several d_sat (window kernel vs the exact kernel)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2112_10591_b200 as ieds  # noqa: E402
from synth.events import WORKLOADS, batch_events  # noqa: E402

wl = WORKLOADS["C3"]
c = wl.scene
xy, off = batch_events(c, wl.seed, 0, 296)
dev = torch.device("cuda", 0)
txy, toff = torch.from_numpy(xy.view(np.int32)).to(dev), torch.from_numpy(off).to(dev)
S = torch.empty((296, c.height, c.width), dtype=torch.float32, device=dev)
res = {}
for d_sat in (6.0, 9.0, 12.0):
    for exact in (False, True):
        with ieds.Builder(c.width, c.height, wl.n_d, wl.n_f, d_sat=d_sat, device=0, exact_edt=exact) as b:
            for _ in range(2):
                b.build_batch(txy, toff, S)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                b.build_batch(txy, toff, S)
            e1.record()
            torch.cuda.synchronize()
            b.sync()
            res[f"d_sat={d_sat} {'exact' if exact else 'window'}"] = 296 * 5 / (e0.elapsed_time(e1) / 1e3)
print(json.dumps(res))
