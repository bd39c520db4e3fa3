#!/bin/bash
# usage (inside gpurun): bash tools/sweep.sh TAG variants/*.so
# runs tools/stage_bench.py for the in-tree library and every variant library
TAG=$1; shift
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}_sweep.jsonl
: > $OUT
timeout 300 python tools/stage_bench.py >> $OUT 2>gpurun_out/${TAG}_sweep_err.log
for so in "$@"; do
  GS_B200_LIB=$so timeout 300 python tools/stage_bench.py >> $OUT 2>>gpurun_out/${TAG}_sweep_err.log
done
echo done
