#!/bin/bash
# Build an A/B variant of librd_gpu.so with extra nvcc defines:
#   tools/build_variant.sh NAME -DRD_GS_QUAD=0 ...   ->  paper_2102_03515_b200/_build/variants/NAME.so
# (select it with RD_GPU_LIB=paper_2102_03515_b200/_build/variants/NAME.so)
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2102_03515_b200"
out=_build/variants/$name
mkdir -p $out
for f in csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
    -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c $f -o $out/$(basename $f .cu).o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _build/variants/$name.so $out/*.o \
  -lcublas -lcusolver -lcudart_static -lrt -ldl -lpthread
