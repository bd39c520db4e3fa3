#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/fz.log
run() { timeout 400 python bench.py --no-cpu-baseline --steps 30 --warmup 5 2>>gpurun_out/fz_err.log | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', d['value'], d['e2e']['value'], d.get('fused_project',{}).get('value'))" >> gpurun_out/fz.log; }
run fuse
GS_TMP_NOFUSE=1 run nofuse
run fuse
GS_TMP_NOFUSE=1 run nofuse
echo done
