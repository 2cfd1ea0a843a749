#!/bin/bash
# warp tournament engine: parity (GPU parity/edge suites + full-size C2/C3/C5), then sweep and replay A/B
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
T=${1:-tour}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/${T}_full.log 2>&1; echo "exit $?" >> gpurun_out/${T}_full.log
tail -3 gpurun_out/${T}_full.log
for v in 1 0 1; do echo "FS_TOUR=$v"; FS_TOUR=$v timeout 300 python tools/prof_sweep.py 4096; done 2>&1 | tee gpurun_out/${T}_sweep.log
for v in 1 0; do echo "FS_TOUR=$v"; FS_TOUR=$v timeout 300 python tools/prof_replay.py c2; done 2>&1 | tee gpurun_out/${T}_replay.log
