#!/bin/bash
# one-rank run of the slab-distributed bench path (NCCL group of 1), then the thread-emulated GPU tests
O=gpurun_out; mkdir -p $O
timeout 600 python bench.py --dist --steps 3 --warmup 3 > $O/d2_bench_dist.json 2> $O/d2_bench_dist.err; echo "dist bench rc=$?"
timeout 600 python bench.py --dist --mode block --steps 3 --warmup 3 > $O/d2_bench_dist_block.json 2> $O/d2_bench_dist_block.err; echo "dist block rc=$?"
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > $O/d2_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/d2_pytest.log; tail -5 $O/d2_bench_dist.err; cat $O/d2_bench_dist.json | head -c 1500
