#!/bin/bash
# like variant_run.sh, with the NEXT rows (f2 simulator time)
for v in "$@"; do
  cp paper_2409_14961_b200/libuellm.so.$v paper_2409_14961_b200/libuellm.so
  timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), 'stats', round(d['stage_ms']['stats'],3), 'f2', round(d['next_rows']['f2_simulate']['ms'],3), d['next_rows']['f2_simulate']['totals']['viol'], d['dp_cost'])"
done
