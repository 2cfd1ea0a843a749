#!/bin/bash
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
for i in 1 2; do
  for t in 6 4 2; do echo "tour $t"; FS_TOUR=$t timeout 300 python tools/prof_replay.py c2; done
  for t in 6 4 2; do echo "tour $t slice512"; FS_TOUR=$t timeout 300 python tools/prof_sweep.py 512; done
done > gpurun_out/tour3.log 2>&1
grep -v '^$' gpurun_out/tour3.log | cut -c1-90
