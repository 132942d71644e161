V=paper_2102_03515_b200/_build/variants
for v in default fA fB fC fD fE; do
  if [ $v = default ]; then L=""; else L="RD_GPU_LIB=$V/$v.so"; fi
  echo "== $v"; env $L timeout 300 python tools/gs_trace.py gpurun_out/trace_$v.txt 2>&1 | grep "^L=127" | head -1 | cut -c1-160
done > gpurun_out/p16_feat.txt 2>&1
