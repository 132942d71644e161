"""Sub-step cycle breakdown of the lattice GS kernel (one tile's thread 0): RD_GS_CTRACE.

usage: python tools/gs_ctrace.py [n] [tile]   (tile -1 = the middle tile)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = "gpurun_out/ctrace.txt"
if os.path.exists(path):
    os.remove(path)
os.environ["RD_GS_CTRACE"] = path
os.environ["RD_GS_CTRACE_TILE"] = sys.argv[2] if len(sys.argv) > 2 else "0"
import torch  # noqa: E402

from paper_2102_03515_b200 import rd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
s = rd.build_system(rd.build_structured_cube(n), 1.0 / n ** 2, "ball")
h = rd.build_amg(s.A)
for l in range(h.num_levels - 1):
    A = h.level(l)
    x = torch.rand(A.rows, dtype=torch.float64, device="cuda")
    f = torch.rand(A.rows, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(2):
        h.level_sweep(l, True, f, x, y)
h.ctx.synchronize()
lines = open(path).read().splitlines()
names = ["halo wait", "loads+C", "B", "waits", "-", "barrier", "->next"]
for i in range(0, len(lines), 2):
    hdr = lines[i].split()
    v = np.array([int(t) for t in lines[i + 1].split()], dtype=np.int64).reshape(-1, 8)[:, :7]
    v = v[5:-5]  # steady state
    nxt = np.roll(v[:, :1], -1, axis=0)
    d = np.diff(np.concatenate([v, nxt], axis=1), axis=1)[:-1]
    med = np.median(d, axis=0)
    print(f"L={hdr[1]} tile {hdr[5]} warp {hdr[7]}: cycles/step median {np.median(np.diff(v[:, 0])):.0f}: " +
          ", ".join(f"{nm} {m:.0f}" for nm, m in zip(names, med)), flush=True)
