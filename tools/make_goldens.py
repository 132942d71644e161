"""Write tests/golden/baseline_configs.json: the CPU oracle's answers at the BASELINE configs.

The reference pins no iteration counts, solutions or error norms at these sizes (SURVEY.md
§8(c)); the oracle's outputs are the goldens.  Per config: PCG iterations and residual history,
||u||_2 and sum(u) of the solution, sample entries, and the error gates -- ||u - u_bar||_L2 with
the target's rule (assembly.cpp:312-331), and l2_error / h1_semi_error (assembly.cpp:265-310) with
the target field as the exact function: ||u - u_bar||_L2 (degree-5 rule) and ||grad(u - u_bar)||_L2
(grad u_bar: oracle Target::grad -- for the smooth target manufactured_exact(0), SURVEY.md §8(f);
for sine+random the sine part plus the P1 interpolant's gradient on the located Kuhn tet).
Configs: C1, the C3 rho sweep, C2, C4 (n = 256), and two non-power-of-two full solves (n = 129
ball, n = 161 smooth: inexact coordinates, no uniform-geometry / uniform-stencil fast paths).
usage: python tools/make_goldens.py   (CPU, several minutes with 8 threads; ~16 GB for C4)
"""
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as O  # noqa: E402

O.build()
O.set_num_threads(os.cpu_count() or 1)
cases = [("C1", 32, 2.0 ** -10, "smooth")]
cases += [(f"C3_rho{rho:g}", 64, rho, "sine_random") for rho in (1.0, 1e-2, 1e-4, 1e-6, 2.0 ** -12)]
cases += [("C2", 128, 2.0 ** -14, "ball")]
cases += [("N129_ball", 129, 1.0 / 129 ** 2, "ball"), ("N161_smooth", 161, 1.0 / 161 ** 2, "smooth")]
cases += [("C4", 256, 2.0 ** -16, "smooth")]
out = {"_source": "tools/make_goldens.py (CPU oracle, oracle/rd_oracle.cpp), tol 1e-8, zero initial guess", "cases": []}
for name, n, rho, target in cases:
    m = O.build_structured_cube(n)
    s = O.build_system(m, rho, target, 0)
    r = O.pcg(s.A, "amg", s.f, 1e-8, 500)
    u = r.x
    idx = [0, len(u) // 3, len(u) // 2, len(u) - 1]
    e = {"name": name, "n": n, "rho": rho, "target": target, "n_dofs": int(len(u)),
         "iterations": int(r.iterations), "residual_history": [float(v) for v in r.residual_history],
         "u_norm2": float(np.linalg.norm(u)), "u_sum": float(np.sum(u)),
         "u_samples": {str(i): float(u[i]) for i in idx},
         "l2_u_minus_target": math.sqrt(O.l2_error_target_squared(m, s, u, target, n, 0))}
    l2d5, h1 = O.error_norms_target(m, s, u, target, n, 0)
    e["l2_deg5_u_minus_target"] = l2d5
    e["h1_u_minus_target"] = h1
    if target == "smooth":  # the same gate through manufactured_exact(0) (c = 1 exactly)
        assert h1 == O.h1_semi_error_manufactured(m, s, u, 0.0)
    out["cases"].append(e)
    print(name, e["iterations"], e["l2_u_minus_target"], flush=True)
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "baseline_configs.json"), "w"), indent=1)
