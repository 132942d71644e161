O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > $O/d1_pytest.log 2>&1; echo "rc=$?" >> $O/d1_pytest.log
tail -30 $O/d1_pytest.log
