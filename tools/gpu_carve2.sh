#!/bin/bash
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
for i in 1 2 3 4; do
  echo "carve default"; timeout 300 python tools/prof_sweep.py 4096
  echo "carve 25"; FS_SWEEP_CARVE=25 timeout 300 python tools/prof_sweep.py 4096
done > gpurun_out/carve2.log 2>&1
grep -v '^$' gpurun_out/carve2.log
