#!/bin/bash
# Round profile: plain run (must exit 0), launch list, one ncu --set full capture of the
# dominant kernels.  usage (via gpurun): bash tools/profile_round.sh TAG
T=${1:-p}; O=gpurun_out; mkdir -p $O
python bench.py --profile --steps 1 --warmup 1 > $O/${T}_plain.json 2>$O/${T}_plain.err || { echo "plain run failed"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/${T}_launches.csv python bench.py --profile --steps 1 --warmup 1 > $O/${T}_ncu1.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"gs_lattice5_kernel|spmv_staged_kernel|coarse_tail_kernel" -c 4 -o $O/${T}_full \
  python bench.py --profile --steps 1 --warmup 0 > $O/${T}_ncu2.log 2>&1; echo "full rc=$?"
ncu -i $O/${T}_full.ncu-rep --page details --csv > $O/${T}_full_details.csv 2>&1
ncu -i $O/${T}_full.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.avg.per_cycle_active > $O/${T}_full_raw.csv 2>&1
echo done
