#!/bin/bash
# session-4 check 3: ACT parity + walk v4 timings; sweep A/B (HEAD lib = A) x4
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "act or test_full_size" > gpurun_out/s4c_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/s4c_pytest.log
tail -2 gpurun_out/s4c_pytest.log
timeout 300 python tools/time_act.py c3 5 both > gpurun_out/s4c_time_act.log 2>&1
grep -A3 'per call' gpurun_out/s4c_time_act.log
for i in 1 2 3 4; do
  echo A; FS_LIB=$PWD/paper_2411_15997_b200/lib/libfairserve_ab.so timeout 300 python tools/prof_sweep.py 4096
  echo B; timeout 300 python tools/prof_sweep.py 4096
done > gpurun_out/s4c_ab_sweep.log 2>&1
cat gpurun_out/s4c_ab_sweep.log
