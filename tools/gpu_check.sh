#!/bin/bash
# One gpurun call: build, smoke, GPU tests, bench line, ncu launch list + full capture.
# usage: gpurun --timeout 1800 -- 'bash tools/gpu_check.sh TAG [skip_tests] [skip_full]'
TAG=${1:-r01}
mkdir -p gpurun_out
exec > >(tee gpurun_out/check_$TAG.log) 2>&1
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()"
if [ "$2" != "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
fi
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
if [ "$3" != "1" ]; then
  # reports stay in /tmp (gpurun_out is capped at 64 MiB); the csv exports come back
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_' -o /tmp/prof_full_$TAG \
     python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-sim > gpurun_out/ncu_full_$TAG.log 2>&1
  tail -3 gpurun_out/ncu_full_$TAG.log
  ncu -i /tmp/prof_full_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$TAG.csv
  ncu -i /tmp/prof_full_$TAG.ncu-rep --page source --csv -k k_dp_tiles > gpurun_out/ncu_src_dp_$TAG.csv 2>&1
  # NEXT-row kernels (f2 simulator, f4 predictor, f3 HELR): first launches of each
  for spec in "sim:k_sim:5" "predict:k_predict:3" "helr:k_helr:23"; do
    IFS=: read name rx cnt <<< "$spec"
    timeout 600 ncu --set full --clock-control none -k regex:"$rx" -c $cnt -o /tmp/prof_${name}_$TAG \
       python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${name}_$TAG.log 2>&1
    ncu -i /tmp/prof_${name}_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${name}_$TAG.csv
  done
  du -sh gpurun_out
fi
ls -la gpurun_out
