O=gpurun_out
bash tools/ab_probe.sh aux1 aux2 > $O/p9_ab.txt 2>&1
RD_GPU_LIB=paper_2102_03515_b200/_build/variants/aux1.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "sweep or gs or vcycle or lattice" > $O/p9_pytest.log 2>&1; echo rc=$? >> $O/p9_pytest.log
