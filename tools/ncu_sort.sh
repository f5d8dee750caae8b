#!/bin/bash
# ncu --set full of the sort-stage kernels of one c4 step (fused reload pack + both scatter passes);
# source-page exports for the SASS attribution.  usage: gpurun -- 'bash tools/ncu_sort.sh TAG'
TAG=${1:-sort}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_reload_pack32|k_sort_down' -c 3 \
   -o /tmp/prof_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-sim --no-configs \
   > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$TAG.csv
ncu -i /tmp/prof_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_details_$TAG.csv
for k in k_reload_pack32 k_sort_down; do
  ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv -k regex:$k --launch-count 1 > gpurun_out/ncu_src_${k}_$TAG.csv 2>/dev/null
done
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv -k regex:k_sort_down --launch-skip 1 --launch-count 1 > gpurun_out/ncu_src_sd1_$TAG.csv 2>/dev/null
ls -la gpurun_out | grep $TAG
