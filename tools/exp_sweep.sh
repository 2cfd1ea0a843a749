#!/bin/bash
# sweep/replay A/B: parity first (tiny + C2 + full-size C5 sweep sample), then timings for the given FS_SWEEP_MINB values
python paper_2411_15997_b200/build.py > /dev/null
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x -k "sweep or replay or step or example or edge or empty or single or filtered or error" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
for m in "$@"; do echo "MINB=$m"; FS_SWEEP_MINB=$m timeout 300 python tools/prof_sweep.py 4096; done
timeout 300 python tools/prof_replay.py c2
