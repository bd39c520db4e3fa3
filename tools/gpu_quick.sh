#!/bin/bash
# usage: gpu_quick.sh TAG [pytest-args]
TAG=$1; shift
/usr/local/graft/bin/gpurun --timeout 900 -- "timeout 400 python -m pytest tests -x -q -m gpu $* > gpurun_out/${TAG}_tests.log 2>&1; echo rc=\$? >> gpurun_out/${TAG}_tests.log; timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1" > gpurun_out/${TAG}_call.txt 2>&1
tail -3 gpurun_out/${TAG}_tests.log
python - <<PY
import json
for l in open("gpurun_out/${TAG}_bench.log"):
    if l.startswith("{"):
        d=json.loads(l); print(d["value"], d["ms_per_step"], d["render_fps"], d["stage_ms"], d["e2e"]["value"])
PY
tail -2 gpurun_out/${TAG}_bench.log | cut -c1-300
