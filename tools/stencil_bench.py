"""Time the lattice stencil SpMV (rd_gpu_spmv on a hierarchy level with stencil facts) with CUDA
events, device vectors, L2 flushed between launches.  usage: RD_GPU_LIB=... python tools/stencil_bench.py [n]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03515_b200 import rd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
s = rd.build_system(rd.build_structured_cube(n), 2.0 ** -14, "ball")
h = rd.build_amg(s.A)
ctx = s.A.ctx
stream = torch.cuda.ExternalStream(rd.lib().rd_gpu_ctx_stream(ctx.h))
flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")  # 256 MB, read (clean lines) to evict L2
for lvl in range(2):
    A = h.level(lvl)
    x = torch.rand(A.rows, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    torch.cuda.synchronize()
    ts = []
    with torch.cuda.stream(stream):
        for it in range(60):
            if it % 2 == 0:
                flush.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ctx.check(rd.lib().rd_gpu_spmv(ctx.h, A.h, x.data_ptr(), y.data_ptr()))
            b.record()
            ts.append((a, b))
    torch.cuda.synchronize()
    cold = sorted(a.elapsed_time(b) * 1e3 for a, b in ts[6::2])
    warm = sorted(a.elapsed_time(b) * 1e3 for a, b in ts[7::2])
    us = cold
    rp, ci, v = A.download()
    ref = rd.spmv(rd.Csr.from_arrays(A.rows, A.cols, rp, ci, v, ctx), x.cpu().numpy())  # CSR kernel
    ok = (y.cpu().numpy() == ref).all()
    print(f"level {lvl} rows {A.rows} stencil={h.stencil_source(lvl)} median {us[len(us)//2]:.2f} us min {us[0]:.2f} "
          f"warm {warm[len(warm)//2]:.2f} ({16 * A.rows / us[len(us)//2] / 1e3:.0f} GB/s of x+y cold)  same_as_csr_path={ok}")
