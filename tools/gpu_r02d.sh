#!/bin/bash
# full GPU suite, then sweep / replay A/B of the engine defaults (FS_TOUR unset) vs the heap-only
# engine (FS_TOUR=0), then the C4 / C3 profile stage times
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
T=${1:-r02d}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
for v in d 0 d 0; do echo "FS_TOUR=$v"; if [ $v = d ]; then timeout 300 python tools/prof_sweep.py 4096; else FS_TOUR=$v timeout 300 python tools/prof_sweep.py 4096; fi; done 2>&1 | tee gpurun_out/${T}_sweep.log
for v in d 0 d 0; do echo "FS_TOUR=$v"; if [ $v = d ]; then timeout 300 python tools/prof_replay.py c2; else FS_TOUR=$v timeout 300 python tools/prof_replay.py c2; fi; done 2>&1 | tee gpurun_out/${T}_replay.log
timeout 300 python tools/time_profile.py c4 5 > gpurun_out/${T}_time_c4.log 2>&1
timeout 300 python tools/time_profile.py c3 5 > gpurun_out/${T}_time_c3.log 2>&1
head -8 gpurun_out/${T}_time_c4.log
