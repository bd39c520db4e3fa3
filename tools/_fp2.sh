#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/stage_bench.py > gpurun_out/fp2_sb.jsonl 2>gpurun_out/fp2_err.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fp2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fp2_tests.log
echo done
