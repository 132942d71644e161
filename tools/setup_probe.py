"""Time the AMG setup pieces (coarsening, Galerkin, hierarchy) on the C2 matrix."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03515_b200 import rd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
s = rd.build_system(rd.build_structured_cube(n), 1.0 / n ** 2, "ball")
A = s.A
for rep in range(2):
    t = time.perf_counter(); flags, P = rd.coarsen_redblack(A); t1 = time.perf_counter()
    Ac = rd.galerkin_coarse(A, P); t2 = time.perf_counter()
    h = rd.build_amg(A); t3 = time.perf_counter()
    m = rd.build_structured_cube(n); s2 = rd.build_system(m, 1.0 / n ** 2, "ball"); s2.ctx.synchronize(); t4 = time.perf_counter()
    print(f"coarsen {1e3*(t1-t):.1f} ms  galerkin {1e3*(t2-t1):.1f} ms  build_amg {1e3*(t3-t2):.1f} ms  mesh+assembly {1e3*(t4-t3):.1f} ms")
