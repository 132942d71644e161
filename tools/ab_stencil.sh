# A/B the lattice stencil SpMV variants (tools/build_variant.sh builds them): correctness, then ncu launch times
for v in ${@:-head}; do
  echo "== $v"
  RD_GPU_LIB=paper_2102_03515_b200/_build/variants/$v.so timeout 300 python tools/stencil_bench.py 128 | grep -o "level.*stencil=[a-z]*\|same_as_csr_path=.*"
  RD_GPU_LIB=paper_2102_03515_b200/_build/variants/$v.so timeout 600 ncu --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:stencil_spmv --launch-skip 56 -c 8 python tools/stencil_bench.py 128 2>/dev/null | grep -E "gpu__time|inst_exec" | awk -F'","' '{print $9, $(NF-2), $NF}' | sort | uniq -c
done
