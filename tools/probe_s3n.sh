V=paper_2102_03515_b200/_build/variants
{
echo "== ls1000"; RD_GPU_LIB=$V/ls1000.so timeout 300 python tools/gs_trace.py gpurun_out/trace_a.txt 2>&1 | grep "^L=127" | head -1 | cut -c1-160
echo "== asleep1000"; RD_GS_ASLEEP=1000 timeout 300 python tools/gs_trace.py gpurun_out/trace_b.txt 2>&1 | grep "^L=127" | head -1 | cut -c1-160
echo "== ls1000+asleep1000"; RD_GS_ASLEEP=1000 RD_GPU_LIB=$V/ls1000.so timeout 300 python tools/gs_trace.py gpurun_out/trace_c.txt 2>&1 | grep "^L=127" | head -1 | cut -c1-160
} > gpurun_out/p17.txt 2>&1
