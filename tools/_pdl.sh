#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pdl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pdl_tests.log
: > gpurun_out/pdl_sb.jsonl
for so in "" variants/nopdl.so "" variants/nopdl.so; do
  GS_B200_LIB=$so timeout 300 python tools/stage_bench.py >> gpurun_out/pdl_sb.jsonl 2>>gpurun_out/pdl_err.log
done
echo done
