O=gpurun_out
python tools/spmv_probe.py > $O/p1_spmv.txt 2>&1
RD_SPMV_NOPROD=1 python tools/spmv_probe.py >> $O/p1_spmv.txt 2>&1
for d in 0 1 2 3 4 8 64 1024; do RD_GS_DEBUG=$d timeout 120 python tools/gs_probe.py 128 >> $O/p1_gs.txt 2>&1; done
timeout 200 python tools/gs_ctrace5.py 128 -1 0 > $O/p1_ctrace.txt 2>&1
timeout 200 python tools/gs_ctrace5.py 128 -1 1 >> $O/p1_ctrace.txt 2>&1
