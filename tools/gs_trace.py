"""Dump per-tile step timestamps of one lattice sweep per level (RD_GS_TRACE)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace.txt"
if os.path.exists(path):
    os.remove(path)
os.environ["RD_GS_TRACE"] = path
from paper_2102_03515_b200 import rd  # noqa: E402

n = 128
s = rd.build_system(rd.build_structured_cube(n), 1.0 / n ** 2, "ball")
h = rd.build_amg(s.A)
import torch  # noqa: E402

for l in range(h.num_levels - 1):
    A = h.level(l)
    x = torch.rand(A.rows, dtype=torch.float64, device="cuda")
    f = torch.rand(A.rows, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(2):
        h.level_sweep(l, True, f, x, y)
h.ctx.synchronize()
# analyse
lines = open(path).read().splitlines()
i = 0
while i < len(lines):
    hdr = lines[i].split()
    L, nty, ntz, ns = int(hdr[1]), int(hdr[3]), int(hdr[5]), int(hdr[7])
    T = np.array([[int(v) for v in lines[i + 1 + t].split()] for t in range(nty * ntz)], dtype=np.int64)
    H = np.array([[int(v) for v in lines[i + 1 + nty * ntz + t].split()] for t in range(nty * ntz)], dtype=np.int64)
    i += 1 + 2 * nty * ntz
    if nty > 1:
        # y crossing tile 0 -> tile 1: upstream step v+16 (lane (0,0) clock), helper commit of v, downstream step v
        v = np.arange(4, ns - 20)
        up, hc, dn = T[0, 2 + v + 16], H[1, 2 + v], T[1, 2 + v]
        print(f"   y crossing 0->1 (ns): upstream step -> halo commit {np.median(hc - up):.0f}, "
              f"commit -> downstream step {np.median(dn - hc):.0f}")
    if ntz > 1:
        v = np.arange(4, ns - 12)
        up, hc, dn = T[0, 2 + v + 8], H[nty, 2 + v], T[nty, 2 + v]
        print(f"   z crossing 0->{nty} (ns): upstream step -> halo commit {np.median(hc - up):.0f}, "
              f"commit -> downstream step {np.median(dn - hc):.0f}")
    t0 = T[:, 0].min()
    start = (T[:, 0] - t0) / 1e3
    steps = (T[:, 2:] - t0) / 1e3
    end = steps[:, -1]
    dt = np.diff(steps, axis=1)
    print(f"L={L} tiles={nty}x{ntz} ns={ns}: span {end.max():.1f} us; start max {start.max():.1f}; "
          f"median step {np.median(dt):.3f} us; p90 step {np.percentile(dt, 90):.3f}; "
          f"tile0 steps {np.median(dt[0]):.3f}; last tile start->first step {steps[-1,0]-start[-1]:.1f}")
    if nty * ntz > 1:
        # lag of each tile's step 0 vs its first-row step, along the diagonal
        print("   first-step time per tile (y fastest):", np.round(steps[:, 0], 1)[: min(24, nty * ntz)])
    if nty * ntz > 1:
        # halo hand-off: tile (y, z) step k needs the (y-1, z) tile's step k + TY - 1 (its last
        # line's row of the same position) and the (y, z-1) tile's step k + TZ - 1
        TY, TZ = 16, 8
        ly, lz = [], []
        for t in range(nty * ntz):
            ty_, tz_ = t % nty, t // nty
            if ty_ > 0:
                o = t - 1
                ly.append(np.median(steps[t, : ns - TY] - steps[o, TY - 1: ns - 1]))
            if tz_ > 0:
                o = t - nty
                lz.append(np.median(steps[t, : ns - TZ] - steps[o, TZ - 1: ns - 1]))
        print(f"   median hand-off lag: y {np.median(ly):.2f} us, z {np.median(lz):.2f} us; "
              f"tile start offsets: mean per y-tile {np.median(np.diff(steps[:nty, 0])):.2f} us, "
              f"per z-tile {np.median(np.diff(steps[::nty, 0])):.2f} us")
