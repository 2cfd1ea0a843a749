#!/bin/bash
# interleaved sweep A/B: A = lib/libfairserve_ab.so, B = the working-tree build; N pairs; optional pytest filter
mkdir -p gpurun_out
T=${1:-ab}; N=${2:-5}; K=${3:-}
python paper_2411_15997_b200/build.py > /dev/null
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
  tail -2 gpurun_out/${T}_pytest.log
fi
for i in $(seq $N); do
  echo A; FS_LIB=$PWD/paper_2411_15997_b200/lib/libfairserve_ab.so timeout 300 python tools/prof_sweep.py 4096
  echo B; timeout 300 python tools/prof_sweep.py 4096
done > gpurun_out/${T}_ab_sweep.log 2>&1
cat gpurun_out/${T}_ab_sweep.log | grep -v '^$'
