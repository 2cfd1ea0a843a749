#!/bin/bash
mkdir -p gpurun_out
T=${1:-s4d}
python paper_2411_15997_b200/build.py > /dev/null
timeout 600 python -m pytest tests -m gpu -x -q -k "act or test_full_size" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
timeout 300 python tools/time_act.py c3 5 both > gpurun_out/${T}_time_act.log 2>&1
grep -A3 'per call' gpurun_out/${T}_time_act.log
