"""Where an rd_gpu_solve_host_mesh call spends its time at n (default 128): wall clock per call
against the setup / solve phases it reports, and the three-call device path beside it."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03515_b200 import rd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ctx = rd.default_context()
mesh = rd.build_structured_cube(n)
rho = 1.0 / n ** 2
xyz, tets, bnd = mesh.download()
px, pt, pb = (torch.from_numpy(a).pin_memory() for a in (xyz, tets, bnd))
u = torch.empty(int((bnd == 0).sum()), dtype=torch.float64).pin_memory()
for _ in range(3):
    rd.solve_host_mesh(px.numpy(), pt.numpy(), pb.numpy(), rho, "ball", 1e-8, u=u, ctx=ctx)
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = rd.solve_host_mesh(px.numpy(), pt.numpy(), pb.numpy(), rho, "ball", 1e-8, u=u, ctx=ctx)
    torch.cuda.synchronize()
    w = 1e3 * (time.perf_counter() - t0)
    print(f"host mesh call {w:.2f} ms: setup {1e3 * out.setup_seconds:.2f} solve {1e3 * out.solve_seconds:.2f} "
          f"rest {w - 1e3 * (out.setup_seconds + out.solve_seconds):.2f}")
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = rd.build_system(mesh, rho, "ball")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    h = rd.build_amg(s.A)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    r = rd.pcg(s.A, "amg", s.f(), 1e-8, 500, hierarchy=h)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"device path: build_system {1e3 * (t1 - t0):.2f} build_amg {1e3 * (t2 - t1):.2f} pcg {1e3 * (t3 - t2):.2f}")
