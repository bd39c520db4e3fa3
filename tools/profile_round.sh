#!/bin/bash
# usage (inside gpurun): bash tools/profile_round.sh TAG
# launch list + ncu --set full of the step's kernels for bench.py (c3), written to gpurun_out/
TAG=$1
mkdir -p gpurun_out
timeout 400 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_tests.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_tests.log
timeout 300 python bench.py --steps 30 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 110 -c 150 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --profile --no-cpu-baseline --steps 4 --warmup 4 \
  > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'blend_|preprocess_|ssim_|onesweep|bucket_|instance_write|window_|depth_hist|tile_ranges' -s 36 -c 24 \
  -o gpurun_out/${TAG}_full -f python bench.py --profile --no-cpu-baseline --steps 2 --warmup 4 \
  > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
