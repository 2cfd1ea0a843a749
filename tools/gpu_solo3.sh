#!/bin/bash
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
for i in 1 2 3; do
  echo "4096 regular"; timeout 300 python tools/prof_sweep.py 4096
  echo "4096 solo16"; FS_SWEEP_SOLO_ALL=1 timeout 300 python tools/prof_sweep.py 4096
done > gpurun_out/solo3.log 2>&1
echo "4096 solo12" >> gpurun_out/solo3.log; FS_SWEEP_SOLO_ALL=1 FS_SWEEP_SOLO_MAX=12 timeout 300 python tools/prof_sweep.py 4096 >> gpurun_out/solo3.log 2>&1
echo "4096 solo20" >> gpurun_out/solo3.log; FS_SWEEP_SOLO_ALL=1 FS_SWEEP_SOLO_MAX=20 timeout 300 python tools/prof_sweep.py 4096 >> gpurun_out/solo3.log 2>&1
echo "4096 solo24" >> gpurun_out/solo3.log; FS_SWEEP_SOLO_ALL=1 FS_SWEEP_SOLO_MAX=24 timeout 300 python tools/prof_sweep.py 4096 >> gpurun_out/solo3.log 2>&1
grep -v '^$' gpurun_out/solo3.log
