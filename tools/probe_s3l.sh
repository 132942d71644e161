O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > $O/p14_pytest.log 2>&1; echo rc=$? >> $O/p14_pytest.log
python bench.py > $O/p14_bench.json 2> $O/p14_bench.err
