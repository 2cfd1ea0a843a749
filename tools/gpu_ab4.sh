#!/bin/bash
# A/B (A = lib/libfairserve_ab.so): the full GPU suite first, then C2 replay, 512 slice, 4096 sweep
mkdir -p gpurun_out
T=${1:-ab4}
python paper_2411_15997_b200/build.py > /dev/null
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
AB=$PWD/paper_2411_15997_b200/lib/libfairserve_ab.so
for i in 1 2; do
  echo A; FS_LIB=$AB timeout 300 python tools/prof_replay.py c2
  echo B; timeout 300 python tools/prof_replay.py c2
  echo A; FS_LIB=$AB timeout 300 python tools/prof_sweep.py 512
  echo B; timeout 300 python tools/prof_sweep.py 512
  echo A; FS_LIB=$AB timeout 300 python tools/prof_sweep.py 4096
  echo B; timeout 300 python tools/prof_sweep.py 4096
done > gpurun_out/${T}_ab.log 2>&1
grep -v '^$' gpurun_out/${T}_ab.log | cut -c1-90
