#!/bin/bash
# sweep vs shared-memory carveout (L1 share): FS_SWEEP_CARVE percent of the SM's 228 KB, -1 = driver default
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
for c in -1 19 -1 19 25 50; do
  if [ "$c" = "-1" ]; then echo "carve default"; timeout 300 python tools/prof_sweep.py 4096
  else echo "carve $c"; FS_SWEEP_CARVE=$c timeout 300 python tools/prof_sweep.py 4096; fi
done > gpurun_out/carve.log 2>&1
cat gpurun_out/carve.log
