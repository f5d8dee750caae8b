#!/bin/bash
# e2e (pipelined host-buffer call) of prebuilt libuellm.so.<variant> builds on c4
for v in "$@"; do
  cp paper_2409_14961_b200/libuellm.so.$v paper_2409_14961_b200/libuellm.so
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sim --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3))"
done
