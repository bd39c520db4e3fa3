#!/bin/bash
# fused next-view projection: GPU tests + bench A/B (inside gpurun)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/fp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fp_tests.log
for mode in 0 1 0 1; do
  GS_BENCH_FUSED_PROJECT=$mode timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('fused=$mode', d['value'], d['e2e']['value'], d['e2e_autograd']['value'], d['stage_ms'], d['roofline']['kernel'], d['roofline']['frac'])" >> gpurun_out/fp_ab.log
done
echo done
