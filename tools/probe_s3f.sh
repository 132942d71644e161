O=gpurun_out
bash tools/ab_probe.sh nopin nolate neither > $O/p6_ab.txt 2>&1
python tools/spmv_probe.py > $O/p6_spmv.txt 2>&1
RD_SPMV_SYNCSTAGE=1 python tools/spmv_probe.py >> $O/p6_spmv.txt 2>&1
