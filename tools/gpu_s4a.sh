#!/bin/bash
# session-4 check: full GPU suite, ACT walk timings (walk vs Jacobi, both cases), C4 profile, ring-cap A/B
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s4a_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/s4a_pytest.log
tail -3 gpurun_out/s4a_pytest.log
( timeout 300 python tools/time_act.py c3 5 both
  FS_ACT_FIXUP=jacobi timeout 300 python tools/time_act.py c3 5 both ) > gpurun_out/s4a_time_act.log 2>&1
grep -A3 'per call' gpurun_out/s4a_time_act.log
timeout 300 python tools/time_profile.py c4 5 > gpurun_out/s4a_time_c4.log 2>&1
head -12 gpurun_out/s4a_time_c4.log
bash tools/gpu_ring.sh
