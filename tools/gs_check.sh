#!/bin/bash
# smoother change check-in: parity suites, then per-level sweep timings
O=gpurun_out; mkdir -p $O; T=${1:-g}
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
tail -4 $O/${T}_pytest.log
timeout 300 python tools/gs_probe.py 128 2>&1 | tail -1
RD_GS_V4=0 timeout 300 python tools/gs_probe.py 64 2>&1 | tail -1
