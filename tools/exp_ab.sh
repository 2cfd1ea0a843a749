#!/bin/bash
# interleaved A/B of the sweep: lib/libfairserve_ab.so (A, e.g. HEAD) vs the working tree build (B)
python paper_2411_15997_b200/build.py > /dev/null
N=${1:-3}
for i in $(seq $N); do
  echo A; FS_LIB=$PWD/paper_2411_15997_b200/lib/libfairserve_ab.so python tools/prof_sweep.py 4096
  echo B; python tools/prof_sweep.py 4096
done
