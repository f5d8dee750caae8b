#!/bin/bash
# ncu --set full of the sort kernels of one c4 step (pack, scatter pass 0, scatter + decode pass 1)
TAG=${1:-sort}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_pack32|k_sort_down|k_sort_up|k_load|k_stats' -c 8 -o gpurun_out/prof_$TAG \
   python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-sim --no-configs > gpurun_out/ncu_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$TAG.csv
for k in DONOTHING; do :; done; exit 0
  ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv -k "regex:${k//[<>, ]/.}" > "gpurun_out/ncu_src_${TAG}_${k//[<>, ]/_}.csv" 2>&1
done
ls -la gpurun_out/*$TAG*
