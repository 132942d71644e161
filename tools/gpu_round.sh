#!/bin/bash
# One GPU check-in: parity suite, bench line, launch list (ncu only after the plain run exits 0).
# usage (via gpurun): bash tools/gpu_round.sh TAG
T=${1:-r}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${T}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; rc=$?
echo "bench rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $O/${T}_launches.csv python bench.py --profile --steps 1 --warmup 1 > $O/${T}_ncu.log 2>&1
  echo "ncu rc=$?"
fi
tail -3 $O/${T}_pytest.log
