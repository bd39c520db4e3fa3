#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/stage_bench.py > gpurun_out/fuse_sb.jsonl 2>gpurun_out/fuse_err.log
timeout 300 python tools/stage_bench.py --n 6000000 --width 3840 --height 2160 >> gpurun_out/fuse_sb.jsonl 2>>gpurun_out/fuse_err.log
echo done
