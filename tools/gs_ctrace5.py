"""Per-warp step timing of the v5 lattice GS kernel (one tile, lane 0 of each warp): RD_GS_CTRACE.

usage: python tools/gs_ctrace5.py [n] [tile] [level]
probes per step (time order): 0 start, 2 old values + leading row terms, 1 fresh values,
3 row sum, 4 x, 5 stores/loads issued.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = "gpurun_out/ctrace5.txt"
if os.path.exists(path):
    os.remove(path)
os.environ["RD_GS_CTRACE"] = path
os.environ["RD_GS_CTRACE_TILE"] = sys.argv[2] if len(sys.argv) > 2 else "0"
only = int(sys.argv[3]) if len(sys.argv) > 3 else -1
import torch  # noqa: E402

from paper_2102_03515_b200 import rd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
s = rd.build_system(rd.build_structured_cube(n), 1.0 / n ** 2, "ball")
h = rd.build_amg(s.A)
for l in range(h.num_levels - 1):
    if only >= 0 and l != only:
        continue
    A = h.level(l)
    x = torch.rand(A.rows, dtype=torch.float64, device="cuda")
    f = torch.rand(A.rows, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    h.level_sweep(l, True, f, x, y)
h.ctx.synchronize()
lines = open(path).read().splitlines()
names = ["box+lead", "fresh wait", "sum", "div", "stores/loads", "->next"]
i = 0
while i < len(lines):
    hdr = lines[i].split()
    ns = int(hdr[3])
    starts = []
    for w in range(4):
        v = np.array([int(t) for t in lines[i + 1 + 2 * w].split()], dtype=np.int64).reshape(-1, 8)[:, [0, 2, 1, 3, 4, 5]]
        v = v[:ns]
        starts.append(v[:, 0])
        vv = v[10:ns - 10]
        if (vv == 0).any():
            print(f"  warp {w}: idle")
            continue
        nxt = np.roll(vv[:, :1], -1, axis=0)
        d = np.diff(np.concatenate([vv, nxt], axis=1), axis=1)[:-1]
        med = np.median(d, axis=0)
        print(f"L={hdr[1]} tile {hdr[5]} warp {w}: cycles/step median {np.median(np.diff(vv[:, 0])):.0f}: " +
              ", ".join(f"{nm} {m:.0f}" for nm, m in zip(names, med)), flush=True)
    base = starts[0]
    for w in range(1, 4):
        if (starts[w][10:ns - 10] != 0).all():
            print(f"   lag of warp {w} behind warp 0 (median cycles): {np.median((starts[w] - base)[10:ns - 10]):.0f}")
    i += 8
