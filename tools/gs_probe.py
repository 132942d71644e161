"""Timing probe for the lattice Gauss-Seidel kernel: per-level sweep times at n
(default 128) with CUDA events on the library stream.  RD_GS_DEBUG selects
diagnostic variants (wrong results, timing only)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03515_b200 import rd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ctx = rd.default_context()
stream = torch.cuda.ExternalStream(ctx.stream)
s = rd.build_system(rd.build_structured_cube(n), 1.0 / n ** 2, "ball")
h = rd.build_amg(s.A)
out = []
for l in range(h.num_levels - 1):
    A = h.level(l)
    x = torch.rand(A.rows, dtype=torch.float64, device="cuda")
    f = torch.rand(A.rows, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        h.level_sweep(l, True, f, x, y)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    R = 20
    for _ in range(R):
        h.level_sweep(l, True, f, x, y)
    b.record(stream)
    torch.cuda.synchronize()
    out.append((l, A.rows, round(a.elapsed_time(b) / R * 1e3, 1), h.stencil_source(l)))
print(os.environ.get("RD_GS_DEBUG", "0"), json.dumps(out))
