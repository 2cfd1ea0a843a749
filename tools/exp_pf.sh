#!/bin/bash
# queue-front prefetch A/B (FS_TOUR bit 8) on the C5 sweep and the C2 replay, interleaved; parity first
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
T=${1:-pf}
FS_TOUR=${SWEEP_ON:-8} timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "sweep or replay" > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
for v in 0 8 0 8; do echo "FS_TOUR=$v"; FS_TOUR=$v timeout 300 python tools/prof_sweep.py 4096; done 2>&1 | tee gpurun_out/${T}_sweep.log
for v in 6 14 6 14; do echo "FS_TOUR=$v"; FS_TOUR=$v timeout 300 python tools/prof_replay.py c2; done 2>&1 | tee gpurun_out/${T}_replay.log
