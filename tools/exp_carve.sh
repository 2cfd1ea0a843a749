#!/bin/bash
# interleaved: default carveout vs FS_SWEEP_CARVE=$1 for the sweep
for i in $(seq ${2:-3}); do
  echo A; python tools/prof_sweep.py 4096
  echo B; FS_SWEEP_CARVE=$1 python tools/prof_sweep.py 4096
done
