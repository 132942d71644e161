O=gpurun_out
timeout 300 python tools/gs_probe.py > $O/p18_gs.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -x > $O/p18_pytest.log 2>&1; echo rc=$? >> $O/p18_pytest.log
bash tools/ab_probe.sh direct0 > $O/p18_ab.txt 2>&1
timeout 300 python tools/gs_trace.py gpurun_out/trace.txt 2>&1 | grep "^L=\|crossing\|lag" | head -8 > $O/p18_trace.txt
