#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_loss.py tests/test_gpu_deterministic.py -m gpu -x -q > gpurun_out/l2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/l2_tests.log
timeout 300 python tools/kernel_probe.py > gpurun_out/l2_probe.log 2>&1
echo done
