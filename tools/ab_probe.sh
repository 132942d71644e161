#!/bin/bash
# A/B of library variants on the lattice sweep probe: tools/ab_probe.sh [variant ...]
V=paper_2102_03515_b200/_build/variants
for r in 1 2; do
  echo "default: $(python tools/gs_probe.py 2>&1 | tail -1)"
  for v in "$@"; do echo "$v: $(RD_GPU_LIB=$V/$v.so python tools/gs_probe.py 2>&1 | tail -1)"; done
done
