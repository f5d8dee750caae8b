#!/bin/bash
# one ncu --set full capture of k_dp_tiles on c4, exported as raw + SASS source csv
TAG=${1:-dp}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dp_tiles -c 1 -o /tmp/prof_$TAG \
   python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-sim > gpurun_out/ncu_$TAG.log 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$TAG.csv
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv > gpurun_out/ncu_src_$TAG.csv 2>&1
ls -la gpurun_out/*_$TAG*
