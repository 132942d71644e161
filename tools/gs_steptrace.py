"""Per-step cycle trace of the lattice sweep (diagnostic build: -DRD_GS_TRACE=1, RD_GPU_LIB=...)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03515_b200 import rd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
lvl = int(sys.argv[2]) if len(sys.argv) > 2 else 0
s = rd.build_system(rd.build_structured_cube(n), 1.0 / n ** 2, "ball")
h = rd.build_amg(s.A)
A = h.level(lvl)
x = torch.rand(A.rows, dtype=torch.float64, device="cuda")
f = torch.rand(A.rows, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    h.level_sweep(lvl, True, f, x, y)
h.ctx.synchronize()
buf = np.zeros((16, 4, 512), dtype=np.uint64)
lib = C.CDLL(rd.LIB_PATH)
rc = lib.rd_gpu_debug_gs_trace(buf.ctypes.data_as(C.c_void_p))
assert rc == 0, rc
T = buf.astype(np.int64)
full = len(sys.argv) > 3
for tile in (0, 1, 2, 8, 9, 15):
    row = []
    for w in range(4):
        t = T[tile, w]
        k = np.nonzero(t)[0]
        d = np.diff(t[k])[8:-8]
        row.append(f"w{w} med {np.median(d):.0f} mean {d.mean():.0f}")
    t = T[tile, 0]
    k = np.nonzero(t)[0]
    d = np.diff(t[k])
    m4 = [round(float(d[8:-8][(np.arange(len(d[8:-8])) + k[9]) % 4 == r].mean())) for r in range(4)]
    print(f"tile {tile:2d}: " + " | ".join(row) + f" | w0 by (s+1)%4 {m4}")
    if full:
        print("  warp0 steps 20..60:", " ".join(str(v) for v in d[20:60]))
cta = np.zeros((16, 4), dtype=np.uint64)
if hasattr(lib, "rd_gpu_debug_gs_trace_cta") and lib.rd_gpu_debug_gs_trace_cta(cta.ctypes.data_as(C.c_void_p)) == 0:
    cta = cta.astype(np.int64)
    for tile in (0, 1, 2, 8, 15):
        t = T[tile, 0]
        k = np.nonzero(t)[0]
        if len(k) == 0:
            continue
        print(f"tile {tile:2d}: prologue {cta[tile, 1] - cta[tile, 0]} cycles, first step end +{t[k[0]] - cta[tile, 1]}, "
              f"steps {t[k[-1]] - t[k[0]]} over {len(k) - 1}, warp-0 end +{cta[tile, 2] - t[k[-1]]} (total {cta[tile, 2] - cta[tile, 0]})")
