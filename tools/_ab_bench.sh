#!/bin/bash
# repeated bench.py runs (stage times), in-tree library and each variant (inside gpurun)
TAG=$1; REPS=${REPS:-2}; shift
for so in "" "$@"; do
  for rep in $(seq $REPS); do
    GS_B200_LIB=$so timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('${so:-intree}', 'gc=${GS_BENCH_GC:-0}', d['value'], d['e2e']['value'], d['stage_ms']['bin_and_sort'], d.get('allocator_during_timed_loops'))" >> gpurun_out/${TAG}_ab.log
  done
done
