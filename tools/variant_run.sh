for v in m4 m3 m4 m3; do
  cp paper_2409_14961_b200/libuellm.so.$v paper_2409_14961_b200/libuellm.so
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sim 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), round(d['stage_ms']['dp_local'],3), d['diagnostics']['dp_candidate_evals'], d['dp_cost'])"
done
