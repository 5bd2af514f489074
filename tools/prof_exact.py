"""One exact-EDT launch (edt_kernel, surfaces + D2) on C3 windows, for an ncu --set full capture."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2112_10591_b200 as ieds
from synth.events import WORKLOADS, batch_events
wl = WORKLOADS['C3']; n = 296
xy, off = batch_events(wl.scene, wl.seed, 0, n)
txy = torch.from_numpy(xy.view(np.int32)).cuda(); toff = torch.from_numpy(off).cuda()
D2 = torch.empty((n, 720, 1280), dtype=torch.int32, device='cuda')
with ieds.Builder(1280, 720, 2, 3, d_sat=6.0, device=0) as b:
    for _ in range(2):
        b.build_batch(txy, toff, sqdist=D2)
    b.sync()
