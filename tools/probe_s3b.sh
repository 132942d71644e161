O=gpurun_out
./tools/fp64lat > $O/p2_lat.txt 2>&1
./tools/stepbench2 > $O/p2_step.txt 2>&1
timeout 200 python tools/gs_trace.py gpurun_out/trace.txt > $O/p2_trace.txt 2>&1
