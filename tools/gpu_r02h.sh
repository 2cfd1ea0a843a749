#!/bin/bash
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "c3 or act" > gpurun_out/r02h_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r02h_pytest.log
tail -3 gpurun_out/r02h_pytest.log
timeout 600 python tools/time_act.py c3 3 2>&1 | head -12 | tee gpurun_out/r02h_time_act_c3.log
