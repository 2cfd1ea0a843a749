#!/bin/bash
# sweep lanes-per-scenario A/B: parity (small + full-size C5 sample) and timing per FS_SWEEP_LPS x FS_SWEEP_MINB
python paper_2411_15997_b200/build.py > /dev/null
for l in "$@"; do
  echo "LPS=$l"
  FS_SWEEP_LPS=$l timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "sweep" 2>&1 | tail -1
  for m in 3 4; do echo "LPS=$l MINB=$m"; FS_SWEEP_LPS=$l FS_SWEEP_MINB=$m timeout 300 python tools/prof_sweep.py 4096; done
done
