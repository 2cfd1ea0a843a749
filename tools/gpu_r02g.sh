#!/bin/bash
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
timeout 600 python tools/time_act.py c3 3 2>&1 | tee gpurun_out/r02g_time_act_c3.log
for s in 512 1024 2048 4096 512; do timeout 300 python tools/prof_sweep.py $s; done 2>&1 | tee gpurun_out/r02g_sweep_slices.log
