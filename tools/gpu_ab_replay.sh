#!/bin/bash
# interleaved A/B of the single replay (A = lib/libfairserve_ab.so, B = working tree)
mkdir -p gpurun_out
T=${1:-abr}
python paper_2411_15997_b200/build.py > /dev/null
AB=$PWD/paper_2411_15997_b200/lib/libfairserve_ab.so
for i in 1 2; do
  echo A; FS_LIB=$AB timeout 300 python tools/prof_replay.py c2
  echo B; timeout 300 python tools/prof_replay.py c2
done > gpurun_out/${T}_ab_replay.log 2>&1
echo A >> gpurun_out/${T}_ab_replay.log; FS_LIB=$AB timeout 300 python tools/prof_replay.py c3 2000000 1 10000 >> gpurun_out/${T}_ab_replay.log 2>&1
echo B >> gpurun_out/${T}_ab_replay.log; timeout 300 python tools/prof_replay.py c3 2000000 1 10000 >> gpurun_out/${T}_ab_replay.log 2>&1
grep -v '^$' gpurun_out/${T}_ab_replay.log | cut -c1-80
