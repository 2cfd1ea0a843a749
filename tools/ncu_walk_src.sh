#!/bin/bash
# source-level stall attribution of the ACT walk (C3, overload always)
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
T=${1:-walk}
timeout 900 ncu --section WarpStateStats --section SourceCounters --import-source on --clock-control none \
  -k regex:'k_act_user_walk' -c 1 -o gpurun_out/${T}_walk python tools/time_act.py c3 1 always > gpurun_out/${T}_walk.log 2>&1
ncu -i gpurun_out/${T}_walk.ncu-rep --page source --csv --print-source cuda > gpurun_out/${T}_walk_src.csv 2>/dev/null
ncu -i gpurun_out/${T}_walk.ncu-rep --page details --csv > gpurun_out/${T}_walk_details.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/${T}_walk_src.csv 70 > gpurun_out/${T}_walk_lines.txt 2>&1
head -75 gpurun_out/${T}_walk_lines.txt
