"""Time the slab-distributed C2 solve with thread-emulated ranks on ONE GPU.

Not a multi-GPU number: every rank shares the device.  It measures what the
distributed driver costs per rank-step (host orchestration, halo copies, the
sequential hand-off of mode exact vs the one-launch pipelined sweep).
usage: python tools/dist_emul_time.py [world ...]
"""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03515_b200 import rd  # noqa: E402
from paper_2102_03515_b200.dist import DeviceOps, DistSolver, ThreadComm  # noqa: E402


def run(world, mode, n=128, reps=3):
    hub = ThreadComm.hub(world)
    times = [None] * world
    its = [None] * world

    def body(rank):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ctx = rd.Context(0, s.cuda_stream)
            ops = DeviceOps(n, 2.0 ** -14, "ball", ctx=ctx)
            solver = DistSolver(ThreadComm(hub, rank), ops, mode=mode)
            solver.pcg(1e-8, 500)
            s.synchronize()
            hub.bar.wait()
            t0 = time.perf_counter()
            for _ in range(reps):
                r = solver.pcg(1e-8, 500)
            s.synchronize()
            hub.bar.wait()
            times[rank] = (time.perf_counter() - t0) / reps
            its[rank] = r.iterations

    th = [threading.Thread(target=body, args=(q,)) for q in range(world)]
    [t.start() for t in th]
    [t.join() for t in th]
    return max(times), its[0]


if __name__ == "__main__":
    worlds = [int(a) for a in sys.argv[1:]] or [1, 2, 4]
    for w in worlds:
        for mode in ("pipelined", "exact", "block"):
            t, it = run(w, mode)
            print(f"world {w} mode {mode:9s}: pcg {1e3 * t:8.2f} ms  ({it} iterations)", flush=True)
