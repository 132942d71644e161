"""Time the V-cycle (and its one-CTA coarse tail) at n: python tools/tail_probe.py [n]."""
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
r = torch.rand(s.n_dofs, dtype=torch.float64, device="cuda")
z = torch.empty_like(r)
for _ in range(3):
    h.apply(r, z)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(stream)
for _ in range(20):
    h.apply(r, z)
b.record(stream)
torch.cuda.synchronize()
print(f"n={n} vcycle {a.elapsed_time(b) / 20 * 1e3:.1f} us  tail={os.environ.get('RD_NO_COARSE_TAIL', '0') == '0'}")
