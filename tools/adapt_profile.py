"""Phase times of one adaptive level on the device (the last, largest level of rdbench adapt's
default run): build_system, AMG setup + PCG, estimate, error norm, dual norm, marking, bisection."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2102_03515_b200 import rd  # noqa: E402

budget = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
ctx = rd.default_context()
t = time.perf_counter()
res = rd.adaptive_solve(rd.build_structured_cube(8), "box", 1e-2, budget)
print(f"adaptive_solve: {time.perf_counter() - t:.3f} s, {len(res.history)} levels, {res.history[-1]['dofs']} dofs")
print("per level s:", [round(r["seconds"], 4) for r in res.history])
m = res.mesh


def tm(name, f, reps=2):
    f()
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = f()
    ctx.synchronize()
    print(f"  {name:28s} {1e3 * (time.perf_counter() - t0) / reps:9.2f} ms")
    return out


print(f"final mesh: {m.n_vertices} vertices, {m.n_tets} tets")
s = tm("build_system", lambda: rd.build_system(m, 1e-2, "box"))
o = tm("solve_system_amg (1e-8)", lambda: rd.solve_system_amg(s.A, s.f(), 1e-8))
print(f"    setup {1e3 * o.setup_seconds:.2f} ms, pcg {1e3 * o.solve_seconds:.2f} ms, {o.iterations} its")
u = o.u
per, g = tm("estimate", lambda: rd.estimate(s, u, "box"))
tm("l2_error_target_squared", lambda: rd.l2_error_target_squared(s, u, "box"))
tm("target_dual_norm", lambda: rd.target_dual_norm(s, u))
mk = tm("mark_dorfler", lambda: rd.mark_dorfler(per, 0.5))
tm("bisect_marked", lambda: rd.bisect_marked(m, mk), reps=1)
h = rd.build_amg(s.A)
print("  levels:", [(h.level(l).rows, h.stencil_source(l)) for l in range(h.num_levels)])

# Gauss-Seidel on the adapted levels: forward sweep time and the lexicographic DAG depth
import torch  # noqa: E402

stream = torch.cuda.ExternalStream(rd.lib().rd_gpu_ctx_stream(ctx.h))
for l in range(h.num_levels - 1):
    A = h.level(l)
    rp, ci, _ = A.download()
    depth = np.zeros(A.rows, np.int64)
    for i in range(A.rows):  # longest chain through lower neighbours
        lo = ci[rp[i]:rp[i + 1]]
        lo = lo[lo < i]
        depth[i] = 1 + (depth[lo].max() if lo.size else 0)
    x = torch.rand(A.rows, dtype=torch.float64, device="cuda")
    f = torch.rand(A.rows, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    with torch.cuda.stream(stream):
        h.level_sweep(l, True, f, x, y)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            h.level_sweep(l, True, f, x, y)
        b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"  level {l}: rows {A.rows:7d} nnz {A.nnz:9d} dag depth {int(depth.max()):6d} fwd sweep {ms:.3f} ms "
          f"({1e3 * ms / depth.max():.2f} us per DAG step)")
