#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_loss.py tests/test_determinism.py -m gpu -x -q > gpurun_out/lc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lc_tests.log
timeout 300 python tools/stage_bench.py > gpurun_out/lc_sb.jsonl 2>gpurun_out/lc_err.log
timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 2>>gpurun_out/lc_err.log | grep '^{' > gpurun_out/lc_bench.json
echo done
