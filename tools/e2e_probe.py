"""Phase timing of the e2e step (host mesh upload -> build_system -> solve -> u to host)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03515_b200 import rd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ctx = rd.Context(0)
mesh = rd.build_structured_cube(n, ctx)
xyz, tets, bnd = mesh.download()
pxyz = torch.from_numpy(xyz).pin_memory()
ptets = torch.from_numpy(tets).pin_memory()
pbnd = torch.from_numpy(bnd).pin_memory()
u_host = torch.empty((n - 1) ** 3, dtype=torch.float64).pin_memory()
u_dev = torch.empty((n - 1) ** 3, dtype=torch.float64, device="cuda")
rho = 1.0 / (n * n)


def tm(fn):
    ctx.synchronize()
    t = time.perf_counter()
    r = fn()
    ctx.synchronize()
    return r, 1e3 * (time.perf_counter() - t)


for it in range(4):
    m, t_up = tm(lambda: rd.mesh_from_arrays(pxyz.numpy(), ptets.numpy(), pbnd.numpy(), ctx))
    s, t_bs = tm(lambda: rd.build_system(m, rho, "ball"))
    o, t_sv = tm(lambda: rd.solve_system_amg(s.A, s.f_ptr, 1e-8, u=u_host))
    _, t_del = tm(lambda: (s.__del__(), m.__del__()))
    s2, t_bs2 = tm(lambda: rd.build_system(mesh, rho, "ball"))
    o2, t_sv2 = tm(lambda: rd.solve_system_amg(s2.A, s2.f_ptr, 1e-8, u=u_dev))
    del s2
    print(f"it {it}: upload {t_up:.1f} build {t_bs:.1f} solve(host u) {t_sv:.1f} free {t_del:.1f} | "
          f"resident: build {t_bs2:.1f} solve {t_sv2:.1f} ms", flush=True)
