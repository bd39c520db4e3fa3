timeout 300 python -m pytest tests/test_gpu_binning.py tests/test_gpu_scale.py -x -q > gpurun_out/g3_tests.log 2>&1; echo rc=$? >> gpurun_out/g3_tests.log
timeout 300 python tools/bin_probe.py > gpurun_out/g3_probe.log 2>&1
timeout 200 python tools/bin_probe.py --n 6000000 --w 3840 --h 2160 >> gpurun_out/g3_probe.log 2>&1
