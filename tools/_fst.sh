#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/fst.jsonl
for so in "" variants/fwd_st8.so variants/fwd_st16.so variants/fwd_st24.so ""; do
  GS_B200_LIB=$so timeout 300 python tools/stage_bench.py >> gpurun_out/fst.jsonl 2>>gpurun_out/fst_err.log
done
echo done
