#!/bin/bash
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k "act or smoke or replay" > gpurun_out/r02e_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r02e_pytest.log
tail -2 gpurun_out/r02e_pytest.log
timeout 600 python tools/exp_combo.py 2>&1 | tee gpurun_out/r02e_combo.log
bash tools/sanitize.sh
