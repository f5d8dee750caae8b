#!/bin/bash
# tile sweep at a query-count override: bash tools/sweep_tile_n.sh CONFIG N TILE...
CFG=$1; N=$2; shift 2
for t in "$@"; do
  timeout 300 python bench.py --config $CFG --queries $N --dp-tile $t --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sim --no-configs > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); s=d['stage_ms']; print('$CFG', $N, $t, round(d['ms_per_step'],3), 'dp', round(s['dp_local'],3), 'casc', round(s['dp_cascade'],3), 'trace', round(s['traceback'],3), d['diagnostics']['tiles'])"
done
