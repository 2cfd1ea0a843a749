#!/bin/bash
# one ncu --set full capture each of k_sweep (S scenarios of the C5 trace) and k_replay (C2), read back here
TAG=${1:-r01b}; S=${2:-1184}
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'^k_sweep' -c 1 -o gpurun_out/${TAG}_sweep \
  python tools/prof_sweep.py $S > gpurun_out/${TAG}_sweep.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'^k_replay$' -c 1 -o gpurun_out/${TAG}_replay \
  python tools/prof_replay.py c2 0 1 > gpurun_out/${TAG}_replay.log 2>&1
python tools/prof_sweep.py $S >> gpurun_out/${TAG}_sweep.log 2>&1
python tools/prof_sweep.py 4096 >> gpurun_out/${TAG}_sweep.log 2>&1
ls -la gpurun_out
