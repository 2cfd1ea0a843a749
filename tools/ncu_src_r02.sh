#!/bin/bash
# source-level instruction / stall attribution: k_sweep over one full wave of C5 scenarios on the
# full 1M-call trace, and the single C2 replay (k_replay_warp)
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
T=${1:-r02s}
timeout 900 ncu --section WarpStateStats --section SourceCounters --import-source on --clock-control none \
  -k regex:'^k_sweep' -c 1 -o gpurun_out/${T}_sweep python tools/prof_sweep.py ${2:-2368} > gpurun_out/${T}_sweep.log 2>&1
ncu -i gpurun_out/${T}_sweep.ncu-rep --page source --csv --print-source cuda > gpurun_out/${T}_sweep_src.csv 2>/dev/null
timeout 600 ncu --section WarpStateStats --section SourceCounters --import-source on --clock-control none \
  -k regex:'k_replay_warp' -c 1 -o gpurun_out/${T}_replay python tools/prof_replay.py c2 0 1 > gpurun_out/${T}_replay.log 2>&1
ncu -i gpurun_out/${T}_replay.ncu-rep --page source --csv --print-source cuda > gpurun_out/${T}_replay_src.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/${T}_sweep_src.csv 60 > gpurun_out/${T}_sweep_lines.txt 2>&1
python tools/ncu_lines.py gpurun_out/${T}_replay_src.csv 60 > gpurun_out/${T}_replay_lines.txt 2>&1
ls -la gpurun_out/
