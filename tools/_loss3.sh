#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/l3_probe.log
for v in 0 1 2 3; do
  GS_B200_LIB=variants/loss_v$v.so timeout 300 python tools/kernel_probe.py 2>/dev/null | tail -1 | sed "s/^/v$v /" >> gpurun_out/l3_probe.log
done
echo done
