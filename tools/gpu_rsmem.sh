#!/bin/bash
# single replay vs its shared-memory budget (the rest of the SM's 256 KB is L1): C3-shaped state (10k users)
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
for kb in -1 128 64 -1 128 64 16; do
  echo "smem budget $kb KB"
  if [ "$kb" = "-1" ]; then timeout 300 python tools/prof_replay.py c3 2000000 1 10000
  else FS_REPLAY_SMEM_KB=$kb timeout 300 python tools/prof_replay.py c3 2000000 1 10000; fi
done > gpurun_out/rsmem.log 2>&1
for kb in -1 128 64; do
  echo "c2 smem budget $kb KB"
  if [ "$kb" = "-1" ]; then timeout 300 python tools/prof_replay.py c2
  else FS_REPLAY_SMEM_KB=$kb timeout 300 python tools/prof_replay.py c2; fi
done >> gpurun_out/rsmem.log 2>&1
grep -v '^$' gpurun_out/rsmem.log
