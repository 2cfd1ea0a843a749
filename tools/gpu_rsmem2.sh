#!/bin/bash
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
for kb in 128 96 160 200 128; do
  echo "kb $kb"; FS_REPLAY_SMEM_KB=$kb timeout 300 python tools/prof_replay.py c2
  echo "kb $kb c3"; FS_REPLAY_SMEM_KB=$kb timeout 300 python tools/prof_replay.py c3 2000000 1 10000
done > gpurun_out/rsmem2.log 2>&1
grep -v '^$' gpurun_out/rsmem2.log | cut -c1-80
