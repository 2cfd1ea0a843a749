#!/bin/bash
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
for i in 1 2; do
  echo "regular"; timeout 300 python tools/prof_sweep.py 4096
  echo "solo8"; FS_SWEEP_SOLO_ALL=1 FS_SWEEP_SOLO_MAX=8 timeout 300 python tools/prof_sweep.py 4096
  echo "solo16"; FS_SWEEP_SOLO_ALL=1 FS_SWEEP_SOLO_MAX=16 timeout 300 python tools/prof_sweep.py 4096
done > gpurun_out/solo4.log 2>&1
grep -v '^$' gpurun_out/solo4.log
