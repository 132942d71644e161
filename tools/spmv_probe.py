"""CSR SpMV timing probe (C2 level-0 A and the level-0 restriction Pt) through the C-ABI
with CUDA events on the library stream.  RD_NO_STENCIL_SPMV=1 forces the CSR kernel on A;
the staged kernel is the cp.async one."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03515_b200 import rd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ctx = rd.default_context()
stream = torch.cuda.ExternalStream(ctx.stream)
s = rd.build_system(rd.build_structured_cube(n), 1.0 / n ** 2, "ball")
h = rd.build_amg(s.A)
out = {}
for name, M in (("A", s.A), ("Pt0", h.level(0, "Pt")), ("P0", h.level(0, "P"))):
    x = torch.rand(M.cols, dtype=torch.float64, device="cuda")
    y = torch.empty(M.rows, dtype=torch.float64, device="cuda")
    call = lambda: rd.lib().rd_gpu_spmv(ctx.h, M.h, x.data_ptr(), y.data_ptr())
    for _ in range(5):
        call()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 50
    a.record(stream)
    for _ in range(R):
        call()
    b.record(stream)
    b.synchronize()
    ms = a.elapsed_time(b) / R
    Z, N = M.nnz, M.rows
    by = 12 * Z + 8 * M.cols + 12 * N + 4
    out[name] = dict(rows=N, nnz=Z, us=ms * 1e3, gbs=by / ms / 1e6)
print(json.dumps(out))
