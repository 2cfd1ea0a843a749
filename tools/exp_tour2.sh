#!/bin/bash
# A/B of the warp-parallel engine pieces (FS_TOUR bits) on the 4096-scenario C5 sweep and the C2 replay,
# then source-level counters of the heap engine on a reduced sweep (100k calls, 1000 users)
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
T=${1:-tour2}
for v in 0 2 4 6 1 0 2; do echo "FS_TOUR=$v"; FS_TOUR=$v timeout 300 python tools/prof_sweep.py 4096; done 2>&1 | tee gpurun_out/${T}_sweep.log
for v in 0 2 4 6; do echo "FS_TOUR=$v"; FS_TOUR=$v timeout 300 python tools/prof_replay.py c2; done 2>&1 | tee gpurun_out/${T}_replay.log
timeout 900 ncu --section WarpStateStats --section SourceCounters --import-source on --clock-control none \
  -k regex:'^k_sweep' -c 1 -o gpurun_out/${T}_sweep python tools/prof_sweep.py 1184 100000 1000 > gpurun_out/${T}_ncu_sweep.log 2>&1
ncu -i gpurun_out/${T}_sweep.ncu-rep --page source --csv --print-source cuda > gpurun_out/${T}_sweep_src.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/${T}_sweep_src.csv 80 > gpurun_out/${T}_sweep_lines.txt 2>&1
head -30 gpurun_out/${T}_sweep_lines.txt
