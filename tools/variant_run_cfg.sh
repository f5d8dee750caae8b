#!/bin/bash
# time prebuilt libuellm.so.<variant> builds on several bench configs (CFGS, default "c5 c4")
for v in "$@"; do
  cp paper_2409_14961_b200/libuellm.so.$v paper_2409_14961_b200/libuellm.so
  for cfg in ${CFGS:-c5 c4}; do
    timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sim --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$cfg', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['stage_ms'].items() if x > 0.01})"
  done
done
