"""Host timing of AMG setup on the C2 system (RD_SETUP_TRACE=1 adds a per-phase breakdown)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03515_b200 import rd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ctx = rd.Context(0)
mesh = rd.build_structured_cube(n, ctx)
s = rd.build_system(mesh, 1.0 / (n * n), "ball")
for it in range(5):
    ctx.synchronize()
    t = time.perf_counter()
    h = rd.build_amg(s.A)
    ctx.synchronize()
    print(f"it {it}: setup {1e3 * (time.perf_counter() - t):.2f} ms, {h.num_levels} levels", flush=True)
    del h
