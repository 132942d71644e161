O=gpurun_out
bash tools/ab_probe.sh hsleep > $O/p8_ab.txt 2>&1
timeout 200 python tools/gs_trace.py gpurun_out/trace.txt > $O/p8_trace.txt 2>&1
