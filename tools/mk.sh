#!/bin/bash
# build the library; non-zero exit on any compile error (for `tools/mk.sh && gpurun ...`)
set -o pipefail
make -s -j8 -C "$(dirname "$0")/../paper_2102_03515_b200" 2>&1 | grep -v "^$" | grep -v "Remark\|warning #20058\|pragma unroll\|^ *\^$\|detected during" | head -30
exit ${PIPESTATUS[0]}
