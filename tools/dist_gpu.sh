#!/bin/bash
# distributed-path GPU tests (thread-emulated ranks, two-process IPC) + emulated timings
O=gpurun_out; mkdir -p $O; T=${1:-d}
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_ipc.py -x -q > $O/${T}_dist.log 2>&1; echo "dist rc=$?" >> $O/${T}_dist.log
tail -25 $O/${T}_dist.log
timeout 600 python tools/dist_emul_time.py 1 2 4 > $O/${T}_emul.txt 2>&1; echo "emul rc=$?"; cat $O/${T}_emul.txt | tail -12
