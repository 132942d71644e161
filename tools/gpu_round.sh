#!/bin/bash
# One GPU check-in: parity suite, bench line (+ the N=1 slab-distributed path), launch list,
# one ncu --set full capture of the dominant kernels (ncu only after the plain runs exit 0).
# usage (via gpurun): bash tools/gpu_round.sh TAG
T=${1:-r}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${T}_smi.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" > $O/${T}_host.txt 2>&1; free -g >> $O/${T}_host.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest.log
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; rc=$?
echo "bench rc=$rc"
timeout 600 python bench.py --dist --steps 3 --warmup 3 --no-e2e > $O/${T}_bench_dist.json 2> $O/${T}_bench_dist.err
echo "bench --dist rc=$?"
if [ $rc -eq 0 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $O/${T}_launches.csv python bench.py --profile --steps 1 --warmup 1 > $O/${T}_ncu.log 2>&1
  echo "ncu launch list rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"gs_lattice5_kernel|spmv_staged_kernel|coarse_tail_kernel|stencil_spmv_tiled_kernel" -c 10 -o $O/${T}_full \
    python bench.py --profile --steps 1 --warmup 0 > $O/${T}_ncu2.log 2>&1; echo "ncu full rc=$?"
  ncu -i $O/${T}_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.avg.per_cycle_active,launch__grid_size,launch__block_size > $O/${T}_full_raw.csv 2>&1
fi
tail -3 $O/${T}_pytest.log
