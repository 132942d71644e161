for cs in 0 32 100 200; do for as in 64 0 16; do
echo "cs $cs as $as: $(RD_GS_CSLEEP=$cs RD_GS_ASLEEP=$as python tools/gs_probe.py 2>&1 | tail -1)"
done; done
