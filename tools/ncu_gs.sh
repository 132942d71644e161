python tools/gs_probe.py 128 > gpurun_out/n1_probe.txt 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gs_lattice5_kernel -s 2 -c 1 -o gpurun_out/n1_gs_uni python tools/gs_probe.py 128 > gpurun_out/n1_ncu.log 2>&1; echo ncu rc=$?
python tools/ncu_stalls.py gpurun_out/n1_gs_uni.ncu-rep 45 > gpurun_out/n1_stalls.txt 2>&1; cat gpurun_out/n1_stalls.txt | head -70
