#!/bin/bash
# Round evidence in one gpurun call: bench line, launch list, one ncu --set full capture of the first
# step's kernels (+ the NEXT-row kernels), the PCIe floor.  Reports stay in /tmp on the box (gpurun_out
# is capped at 64 MiB); the csv exports come back.
# usage: gpurun --timeout 3000 -- 'bash tools/gpu_evidence.sh r02'
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err
timeout 300 python tools/pcie_floor.py > gpurun_out/pcie_$TAG.json 2>&1; cat gpurun_out/pcie_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-configs > /dev/null 2>&1
# the first step's kernels (sync load -> schedule -> stats): about 30 launches
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_' -c 32 -o /tmp/prof_full_$TAG \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-sim --no-configs > gpurun_out/ncu_full_$TAG.log 2>&1
tail -2 gpurun_out/ncu_full_$TAG.log
ncu -i /tmp/prof_full_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$TAG.csv
ncu -i /tmp/prof_full_$TAG.ncu-rep --page source --csv -k regex:k_dp_tiles > gpurun_out/ncu_src_dp_$TAG.csv 2>/dev/null
ncu -i /tmp/prof_full_$TAG.ncu-rep --page source --csv -k regex:k_sort_down --launch-count 1 > gpurun_out/ncu_src_sd0_$TAG.csv 2>/dev/null
ncu -i /tmp/prof_full_$TAG.ncu-rep --page source --csv -k regex:k_sort_down --launch-skip 1 --launch-count 1 > gpurun_out/ncu_src_sd1_$TAG.csv 2>/dev/null
# NEXT-row kernels (f1 Alg. 1, f2 simulator, f3 HELR, f4 predictor): first launch of each
timeout 900 ncu --set full --clock-control none -k regex:'k_alg1_next|k_a1_|k_helr_level|k_sim_|k_pred_' -c 40 -o /tmp/prof_next_$TAG \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/ncu_next_$TAG.log 2>&1
ncu -i /tmp/prof_next_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_next_$TAG.csv
du -sh gpurun_out; ls -la gpurun_out | grep $TAG
