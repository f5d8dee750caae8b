#!/bin/bash
# sort window-group sweep on c4 (bench stage times), one line per setting
mkdir -p gpurun_out
for q in 100000000 8388608 4194304 2097152 1048576; do
  UELLM_SORT_GROUP_Q=$q timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sim > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print($q, round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})"
done | tee gpurun_out/sweep_sort.txt
