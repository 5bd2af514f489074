#!/usr/bin/env python
"""One workload's launch pair for ncu (profiles/r02_ncu_configs.md): builds `windows` windows of a
BASELINE config (C2, C3, C5; events cycled through a pool of distinct generated windows, as bench.py
does) with an optional output format, `warmup` + 1 times, so that
`ncu -k regex:"frame_kernel|window_kernel" -s <2 * warmup> -c 2 python tools/ncu_config.py C2`
captures one steady-state frame and window launch.  Also prints the per-kernel CUDA-event times
of a profiled run (no ncu) for the same batch, and the pixels per launch, so lane-instructions per
pixel can be read off the capture: inst_executed * 32 / pixels.

usage: python tools/ncu_config.py NAME [windows] [out: f32|u8|f16] [warmup]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2112_10591_b200 as ieds  # noqa: E402
from synth.events import WORKLOADS  # noqa: E402


def main():
    name = sys.argv[1]
    wl = WORKLOADS[name]
    c = wl.scene
    nwin = int(sys.argv[2]) if len(sys.argv) > 2 else wl.n_windows
    out = sys.argv[3] if len(sys.argv) > 3 else "f32"
    warmup = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    dev = torch.device("cuda", 0)
    txy, toff, n_ev, pool = bench.cycled_batch(name, 0, nwin, min(nwin, 1000 if name != "C5" else 256), dev)
    dt = {"f32": torch.float32, "u8": torch.uint8, "f16": torch.float16}[out]
    S = torch.empty((nwin, c.height, c.width), dtype=dt, device=dev)
    with ieds.Builder(c.width, c.height, wl.n_d, wl.n_f, d_sat=wl.d_sat, device=0, out=out) as b:
        for _ in range(warmup):
            b.build_batch(txy, toff, S)
        b.sync()
        b.profile(True)
        b.profile_read()
        b.build_batch(txy, toff, S)
        b.sync()
        p = b.profile_read()
    print(f"{name} {out}: {nwin} windows, {n_ev} events, {nwin * c.width * c.height} pixels per launch; "
          f"frame {p['frame'][0]:.4f} ms, window {p['edt'][0]:.4f} ms (CUDA events)")


if __name__ == "__main__":
    main()
