#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_loss.py tests/test_gpu_deterministic.py -m gpu -x -q > gpurun_out/lp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lp_tests.log
timeout 300 python tools/kernel_probe.py > gpurun_out/lp_probe.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ssim|loss_final" -c 3 -o gpurun_out/lp_ssim python tools/stage_bench.py > gpurun_out/lp_ncu.log 2>&1
echo done
