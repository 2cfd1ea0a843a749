#!/bin/bash
# per-line stall attribution of the single replay (k_replay_warp, C2 shape, 200k calls) and of the
# sweep (k_sweep, 592 C5 scenarios on the full trace: one wave of 4 per SM)
mkdir -p gpurun_out
T=${1:-rl}
python paper_2411_15997_b200/build.py > /dev/null
timeout 900 ncu --section WarpStateStats --section SourceCounters --import-source on --clock-control none \
  -k regex:'k_replay_warp' -c 1 -o gpurun_out/${T}_replay python tools/prof_replay.py c2 200000 1 > gpurun_out/${T}_replay.log 2>&1
ncu -i gpurun_out/${T}_replay.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${T}_replay_src.csv 2>/dev/null
python tools/ncu_src_lines.py gpurun_out/${T}_replay_src.csv 60 > gpurun_out/${T}_replay_lines.txt
head -40 gpurun_out/${T}_replay_lines.txt
