#!/bin/bash
# ACT fixup walk: parity (tiny + C2-shape + sharded + full-size) and C3 / C2 timings, A/B vs the Jacobi fixup
mkdir -p gpurun_out
T=${1:-walk}
python paper_2411_15997_b200/build.py > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q -k "act or test_full_size" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
timeout 300 python tools/time_act.py c3 5 always > gpurun_out/${T}_time_act.log 2>&1
FS_ACT_FIXUP=jacobi timeout 300 python tools/time_act.py c3 5 always >> gpurun_out/${T}_time_act.log 2>&1
timeout 300 python tools/time_act.py c3 5 replay >> gpurun_out/${T}_time_act.log 2>&1
cat gpurun_out/${T}_time_act.log
