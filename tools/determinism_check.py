"""Repeat a full build + setup + solve and compare u bit for bit with the first run (a race in
the programmatic-dependent-launch chain or the tile hand-offs would show up as a difference).
usage: python tools/determinism_check.py [n] [repeats]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03515_b200 import rd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
mesh = rd.build_structured_cube(n)
rho = 1.0 / n ** 2
ref = None
for k in range(reps):
    s = rd.build_system(mesh, rho, "ball")
    out = rd.solve_system_amg(s.A, s.f(), 1e-8)
    if ref is None:
        ref = (out.u.copy(), out.iterations)
    else:
        assert out.iterations == ref[1], (k, out.iterations, ref[1])
        assert np.array_equal(out.u, ref[0]), f"run {k} differs from run 0"
print(f"n={n}: {reps} runs bit-identical, {ref[1]} iterations")
