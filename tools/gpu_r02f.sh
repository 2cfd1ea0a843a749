#!/bin/bash
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
T=${1:-r02f}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py -q -x -k "profile or smoke or sweep_small" > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
for r in 512 256 512 256; do echo "FS_WP_R=$r"; FS_WP_R=$r timeout 300 python tools/time_profile.py c4 5 | head -12; done 2>&1 | tee gpurun_out/${T}_time_c4.log
FS_WP_R=256 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "profile" 2>&1 | tail -2
