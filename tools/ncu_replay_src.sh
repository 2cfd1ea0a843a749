#!/bin/bash
# source-level stall/instruction counters of the single replay on a reduced C2 trace
python paper_2411_15997_b200/build.py > /dev/null
timeout 600 ncu --section WarpStateStats --section SourceCounters --import-source on --clock-control none \
  -k regex:'k_replay_warp' -c 1 -o gpurun_out/${1:-r01k}_replay python tools/prof_replay.py c2 100000 1 > gpurun_out/${1:-r01k}_replay.log 2>&1
