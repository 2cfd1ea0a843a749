#!/bin/bash
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
for S in 1024 2048; do
  echo "$S regular"; FS_SWEEP_SOLO=0 timeout 300 python tools/prof_sweep.py $S
  echo "$S solo"; FS_SWEEP_SOLO_MAX=16 timeout 300 python tools/prof_sweep.py $S
done > gpurun_out/solo2.log 2>&1
echo "4096 solo" >> gpurun_out/solo2.log; FS_SWEEP_SOLO_MAX=32 timeout 300 python tools/prof_sweep.py 4096 >> gpurun_out/solo2.log 2>&1
echo "592 solo" >> gpurun_out/solo2.log; timeout 300 python tools/prof_sweep.py 592 >> gpurun_out/solo2.log 2>&1
echo "592 regular" >> gpurun_out/solo2.log; FS_SWEEP_SOLO=0 timeout 300 python tools/prof_sweep.py 592 >> gpurun_out/solo2.log 2>&1
grep -v '^$' gpurun_out/solo2.log
