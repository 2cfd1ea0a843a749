#!/bin/bash
# sweep A/B: parity first, then timings for the FS_SWEEP_MINB values given
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "sweep or replay or step" 2>&1 | tail -3
for m in "$@"; do echo "MINB=$m"; FS_SWEEP_MINB=$m timeout 300 python tools/prof_sweep.py 4096; done
timeout 300 python tools/prof_replay.py c2
