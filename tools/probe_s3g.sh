O=gpurun_out
V=paper_2102_03515_b200/_build/variants
for v in default b8 b4 c256 c256b8; do
  if [ $v = default ]; then echo "$v $(python tools/spmv_probe.py 2>&1|tail -1)"; else echo "$v $(RD_GPU_LIB=$V/$v.so python tools/spmv_probe.py 2>&1|tail -1)"; fi
done > $O/p7_spmv.txt
timeout 200 python tools/gs_trace.py gpurun_out/trace.txt > $O/p7_trace.txt 2>&1
