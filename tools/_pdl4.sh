#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/pdl5.log
run() { timeout 400 python bench.py --no-cpu-baseline --steps 30 --warmup 5 2>>gpurun_out/pdl5_err.log | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', d['value'], d['stage_timed_loop']['value'], d['e2e']['value'], d.get('fused_project',{}).get('value'), d['stage_ms'], d.get('allocator_during_timed_loops'))" >> gpurun_out/pdl5.log; }
run paced
run paced
run paced
echo done
