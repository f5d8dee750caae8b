#!/bin/bash
# one ncu --set full capture of the SEG-DP kernel (k_dp_tiles<V>) on a bench config, exported as raw
# + SASS source csv, the report itself copied back to gpurun_out/
TAG=${1:-dp}
CONFIG=${2:-c4}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dp_tiles -c 1 -o gpurun_out/prof_$TAG \
   python bench.py --config $CONFIG --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-sim --no-configs > gpurun_out/ncu_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$TAG.csv
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv > gpurun_out/ncu_src_$TAG.csv 2>&1
ls -la gpurun_out/*_$TAG*
