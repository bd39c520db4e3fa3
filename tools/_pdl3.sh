#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/pdl3.log
run() { timeout 400 python bench.py --no-cpu-baseline --steps 30 --warmup 5 2>>gpurun_out/pdl3_err.log | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', d['value'], d['stage_timed_loop']['value'], d['e2e']['value'], d.get('fused_project',{}).get('value'), d['stage_ms'])" >> gpurun_out/pdl3.log; }
run pdl_on
GS_PDL_LAUNCH=0 run pdl_off
GS_B200_LIB=variants/notrig.so run notrigger
run pdl_on
GS_PDL_LAUNCH=0 run pdl_off
echo done
