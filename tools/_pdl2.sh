#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pdl2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pdl2_tests.log
timeout 300 python tools/stage_bench.py > gpurun_out/pdl2_sb.jsonl 2>>gpurun_out/pdl2_err.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 2>>gpurun_out/pdl2_err.log | grep '^{' >> gpurun_out/pdl2_bench.jsonl
done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/pdl2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/pdl2_smoke.log
echo done
