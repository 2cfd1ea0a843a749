#!/bin/bash
# strong-scaling slices: sweep of 512 / 1024 C5 scenarios with the solo-slot kernel vs the regular one; parity
mkdir -p gpurun_out
T=${1:-solo}
python paper_2411_15997_b200/build.py > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "sweep" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
for i in 1 2; do
  echo "512 regular"; FS_SWEEP_SOLO=0 timeout 300 python tools/prof_sweep.py 512
  echo "512 solo"; timeout 300 python tools/prof_sweep.py 512
done > gpurun_out/${T}_slices.log 2>&1
echo "296 solo (2 per SM)" >> gpurun_out/${T}_slices.log; timeout 300 python tools/prof_sweep.py 296 >> gpurun_out/${T}_slices.log 2>&1
echo "296 regular" >> gpurun_out/${T}_slices.log; FS_SWEEP_SOLO=0 timeout 300 python tools/prof_sweep.py 296 >> gpurun_out/${T}_slices.log 2>&1
grep -v '^$' gpurun_out/${T}_slices.log
