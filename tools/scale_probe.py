"""One full solve at n (C4 n=256, C5 n=512) on one GPU: phase times, iterations, peak memory.
usage: python tools/scale_probe.py n [target]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03515_b200 import rd  # noqa: E402

n = int(sys.argv[1])
target = sys.argv[2] if len(sys.argv) > 2 else "smooth"
rho = 1.0 / n ** 2
ctx = rd.default_context()
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mesh = rd.build_structured_cube(n, ctx)
    ctx.synchronize()
    t1 = time.perf_counter()
    s = rd.build_system(mesh, rho, target)
    ctx.synchronize()
    t2 = time.perf_counter()
    u = torch.empty(s.n_dofs, dtype=torch.float64, device="cuda")
    out = rd.solve_system_amg(s.A, s.f_ptr, 1e-8, u=u)
    t3 = time.perf_counter()
    free, total = torch.cuda.mem_get_info()
    print(f"n={n} dofs={s.n_dofs} mesh {1e3*(t1-t0):.1f} ms build {1e3*(t2-t1):.1f} ms setup {1e3*out.setup_seconds:.1f} ms "
          f"solve {1e3*out.solve_seconds:.1f} ms iterations {out.iterations} conv {out.converged} "
          f"dof_iters/s {s.n_dofs*out.iterations/(t3-t1):.3e} used {(total-free)/2**30:.1f} GiB", flush=True)
    del s, mesh, u
