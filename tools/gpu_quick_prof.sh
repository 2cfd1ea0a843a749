#!/bin/bash
# profile parity (GPU tests matching "profile") + C4 / C3 profile stage times
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
T=${1:-qp}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py -q -x -k "profile" > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
timeout 300 python tools/time_profile.py c4 5 2>&1 | head -16 | tee gpurun_out/${T}_time_c4.log
timeout 300 python tools/time_profile.py c3 5 2>&1 | head -6 | tee gpurun_out/${T}_time_c3.log
