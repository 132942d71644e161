bash tools/ab_probe.sh hb1 hb2 hb3 hb4 hb5 hb6 > gpurun_out/p4_hb.txt 2>&1
