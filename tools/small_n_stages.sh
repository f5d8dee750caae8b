#!/bin/bash
# stage times of the device-resident step at window-group sizes (c4 shape)
for q in 1000000 3000000 7000000 12500000 25000000; do
  timeout 300 python bench.py --queries $q --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sim > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print($q, round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})"
done
