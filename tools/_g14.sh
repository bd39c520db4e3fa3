timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/g14_bench.log 2>&1
timeout 600 python -m pytest tests/test_multirank_gpu.py -q -x > gpurun_out/g14_mr.log 2>&1; echo rc=$? >> gpurun_out/g14_mr.log
