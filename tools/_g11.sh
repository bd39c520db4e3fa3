timeout 900 python -m pytest tests/test_gpu_benchconfigs.py tests/test_gpu_parity.py tests/test_gpu_scale.py -q > gpurun_out/g11_tests.log 2>&1; echo rc=$? >> gpurun_out/g11_tests.log
timeout 300 python tools/kernel_probe.py > gpurun_out/g11_probe.log 2>&1
