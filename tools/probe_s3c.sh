O=gpurun_out
for as in 64 0 16 256; do echo "as $as: $(RD_GS_ASLEEP=$as python tools/gs_probe.py 2>&1 | tail -1)"; done > $O/p3_sleep.txt 2>&1
bash tools/ab_probe.sh hb4 hb16 > $O/p3_hb.txt 2>&1
