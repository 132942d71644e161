#!/bin/bash
# RD_GS_DEBUG attribution of the lattice sweep time (timing probes; results are wrong):
# 1 no ring waits / backpressure, 2 no box chunk waits, 4 no x stores, 8 no box reads,
# 16 constant stencil, 32 no ring publish, 128 no box warp, 256 no helper warp,
# 512 speculative division (as in production)
for d in ${@:-0 1 4 16 20 138 142 158 394 398 414 415}; do
  echo "dbg $d: $(RD_GS_DEBUG=$d timeout 100 python tools/gs_probe.py 2>&1 | tail -1)"
done
