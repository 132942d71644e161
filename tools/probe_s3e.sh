O=gpurun_out
python tools/gs_probe.py > $O/p5_gs.txt 2>&1
python tools/spmv_probe.py > $O/p5_spmv.txt 2>&1
RD_SPMV_NOPROD=1 python tools/spmv_probe.py >> $O/p5_spmv.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/p5_pytest.log 2>&1; echo rc=$? >> $O/p5_pytest.log
