#!/bin/bash
# FWI sweep specialisation: parity (sweep tests incl. the full 4096-scenario C5 goldens), interleaved A/B
# (FS_SWEEP_FWI=0 vs 1, same library); ACT walk timing
mkdir -p gpurun_out
T=${1:-s4e}
python paper_2411_15997_b200/build.py > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "sweep or act" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
for i in 1 2 3 4; do
  echo A-generic; FS_SWEEP_FWI=0 timeout 300 python tools/prof_sweep.py 4096
  echo B-fwi; timeout 300 python tools/prof_sweep.py 4096
done > gpurun_out/${T}_ab_sweep.log 2>&1
cat gpurun_out/${T}_ab_sweep.log
timeout 300 python tools/time_act.py c3 5 always > gpurun_out/${T}_time_act.log 2>&1
grep -A3 'per call' gpurun_out/${T}_time_act.log
