#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do
timeout 400 python bench.py 2>>gpurun_out/b3_err.log | grep '^{' >> gpurun_out/b3_bench.jsonl
done
timeout 300 python bench.py --impl reference 2>>gpurun_out/b3_err.log | grep '^{' >> gpurun_out/b3_ref.jsonl
echo done
