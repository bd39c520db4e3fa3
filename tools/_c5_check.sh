#!/bin/bash
# c5 regression check: stage timings at 6M/4K for the in-tree lib and variants, then c5 twice
mkdir -p gpurun_out
OUT=gpurun_out/c5chk_sweep.jsonl; : > $OUT
for so in "" variants/oldbin.so variants/oldfwd.so; do
  GS_B200_LIB=$so timeout 300 python tools/stage_bench.py --n 6000000 --width 3840 --height 2160 >> $OUT 2>>gpurun_out/c5chk_err.log
done
timeout 300 python tools/stage_bench.py >> $OUT 2>>gpurun_out/c5chk_err.log
timeout 600 python tools/bench_configs.py --configs c5,c5 --out gpurun_out/c5chk_configs.jsonl > /dev/null 2>>gpurun_out/c5chk_err.log
echo done
