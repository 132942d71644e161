"""Debug: one forward / backward lattice GS pass vs a plain Python restatement."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
from paper_2102_03515_b200 import rd  # noqa: E402
import pyoracle as O  # noqa: E402


def gs_pass(rp, ci, v, f, x, fwd):
    x = x.copy()
    n = len(f)
    order = range(n) if fwd else range(n - 1, -1, -1)
    for i in order:
        s = f[i]
        d = 0.0
        for k in range(rp[i], rp[i + 1]):
            if ci[k] == i:
                d = v[k]
            else:
                s -= v[k] * x[ci[k]]
        x[i] = s / d
    return x


for n in [int(a) for a in sys.argv[1:]] or [3, 4, 8]:
    os_ = O.build_system(O.build_structured_cube(n), 2.0 ** -8, "smooth")
    A = rd.Csr.from_arrays(os_.A.rows, os_.A.cols, os_.A.rp, os_.A.ci, os_.A.v)
    f = O.pseudo_random_vec(A.rows, 1)
    u = O.pseudo_random_vec(A.rows, 2)
    # the level-0 sweep of a 1-level "hierarchy" would not be structured; use sgs_sweep pieces:
    out = rd.sgs_sweep(A, f, u)
    ref_f = gs_pass(os_.A.rp, os_.A.ci, os_.A.v, f, u, True)
    ref = gs_pass(os_.A.rp, os_.A.ci, os_.A.v, f, ref_f, False)
    bad = np.nonzero(out != ref)[0]
    print(f"n={n} rows={A.rows} mismatches={bad.size} first={bad[:10]} dev={out[bad[:3]]} ref={ref[bad[:3]]}")
