#!/bin/bash
# per-step time of the single-tile level (L=8) and the level-0 offsets under RD_GS_DEBUG variants
for d in ${@:-512 513 514 516 520 528 544 640 768 896 1023}; do
  echo "dbg $d: $(RD_GS_DEBUG=$d timeout 60 python tools/gs_trace.py 2>&1 | grep -E '^L=(8|127) ' | sed -E 's/span [^;]*; //; s/start max [^;]*; //' | tr '\n' ' ')"
done
