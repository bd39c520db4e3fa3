#!/bin/bash
# usage (inside gpurun): bash tools/_r2_final.sh TAG -- tests, bench, launch list, ncu full, other configs
TAG=$1
bash tools/profile_round.sh $TAG
timeout 900 python tools/bench_configs.py --configs c2,c4,c5,c5s --out gpurun_out/${TAG}_configs.jsonl > gpurun_out/${TAG}_configs.log 2>&1
timeout 300 python tools/kernel_probe.py > gpurun_out/${TAG}_probe.log 2>&1
