bash tools/ab_probe.sh ls100 ls300 ls1000 > gpurun_out/p11_ab.txt 2>&1
