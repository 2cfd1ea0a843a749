#!/bin/bash
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
for i in 1 2 3; do
  echo "minb 4"; timeout 300 python tools/prof_sweep.py 4096
  echo "minb 5"; FS_SWEEP_MINB=5 timeout 300 python tools/prof_sweep.py 4096
  echo "minb 5 carve 33"; FS_SWEEP_MINB=5 FS_SWEEP_CARVE=33 timeout 300 python tools/prof_sweep.py 4096
done > gpurun_out/minb.log 2>&1
grep -v '^$' gpurun_out/minb.log
