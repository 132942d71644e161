O=gpurun_out
bash tools/ab_probe.sh r32 > $O/p10_ab.txt 2>&1
python tools/spmv_probe.py > $O/p10_spmv.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/p10_pytest.log 2>&1; echo rc=$? >> $O/p10_pytest.log
bash tools/gpu_round.sh s3c
