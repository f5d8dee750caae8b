#!/bin/bash
for t in 0 3584 5632 6144 7168; do
  timeout 300 python bench.py --dp-tile $t --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sim > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print($t, round(d['ms_per_step'],3), round(d['stage_ms']['dp_local'],3), d['diagnostics']['tiles'], d['diagnostics']['fixup_positions'], d['diagnostics']['cascade_reruns'])"
done
