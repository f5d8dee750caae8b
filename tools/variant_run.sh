#!/bin/bash
# time prebuilt libuellm.so.<variant> builds on c4 (stage ms + the DP optimum as a sanity check)
for v in "$@"; do
  cp paper_2409_14961_b200/libuellm.so.$v paper_2409_14961_b200/libuellm.so
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sim ${VR_ARGS:---no-configs} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items() if v > 0.01}, d['dp_cost'])"
done
