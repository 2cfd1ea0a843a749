#!/bin/bash
# interleaved A/B (A = lib/libfairserve_ab.so, B = working tree) of the sweep, the C2 replay and a
# C3-shaped replay; parity first
mkdir -p gpurun_out
T=${1:-ab2}
python paper_2411_15997_b200/build.py > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "replay or sweep or step" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
AB=$PWD/paper_2411_15997_b200/lib/libfairserve_ab.so
for i in 1 2 3; do
  echo A; FS_LIB=$AB timeout 300 python tools/prof_replay.py c2
  echo B; timeout 300 python tools/prof_replay.py c2
done > gpurun_out/${T}_ab_replay.log 2>&1
for i in 1 2; do
  echo A; FS_LIB=$AB timeout 300 python tools/prof_replay.py c3 2000000 1 10000
  echo B; timeout 300 python tools/prof_replay.py c3 2000000 1 10000
done >> gpurun_out/${T}_ab_replay.log 2>&1
grep -v '^$' gpurun_out/${T}_ab_replay.log
for i in 1 2 3 4; do
  echo A; FS_LIB=$AB timeout 300 python tools/prof_sweep.py 4096
  echo B; timeout 300 python tools/prof_sweep.py 4096
done > gpurun_out/${T}_ab_sweep.log 2>&1
grep -v '^$' gpurun_out/${T}_ab_sweep.log
