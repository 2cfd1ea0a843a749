#!/bin/bash
# session-4 check 2: full GPU suite, ACT walk v3 timings, A/B (HEAD lib = A) of the sweep and the C2 replay
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s4b_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/s4b_pytest.log
tail -3 gpurun_out/s4b_pytest.log
timeout 300 python tools/time_act.py c3 5 both > gpurun_out/s4b_time_act.log 2>&1
grep -A4 'per call' gpurun_out/s4b_time_act.log
for i in 1 2 3; do
  echo A; FS_LIB=$PWD/paper_2411_15997_b200/lib/libfairserve_ab.so timeout 300 python tools/prof_sweep.py 4096
  echo B; timeout 300 python tools/prof_sweep.py 4096
done > gpurun_out/s4b_ab_sweep.log 2>&1
cat gpurun_out/s4b_ab_sweep.log
for i in 1 2; do
  echo A; FS_LIB=$PWD/paper_2411_15997_b200/lib/libfairserve_ab.so timeout 300 python tools/prof_replay.py c2
  echo B; timeout 300 python tools/prof_replay.py c2
done > gpurun_out/s4b_ab_replay.log 2>&1
cat gpurun_out/s4b_ab_replay.log
