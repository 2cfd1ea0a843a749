#!/bin/bash
# A/B (A = lib/libfairserve_ab.so) of the C4 profile (per-kernel times); profile parity first
mkdir -p gpurun_out
T=${1:-abc4}
python paper_2411_15997_b200/build.py > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "profile or c4" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
AB=$PWD/paper_2411_15997_b200/lib/libfairserve_ab.so
for i in 1 2; do
  echo A; FS_LIB=$AB timeout 300 python tools/time_profile.py c4 5 | head -8
  echo B; timeout 300 python tools/time_profile.py c4 5 | head -8
done > gpurun_out/${T}_ab.log 2>&1
cat gpurun_out/${T}_ab.log
