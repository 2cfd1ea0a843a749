#!/bin/bash
# interleaved A/B of the C4 profile step: lib/libfairserve_ab.so (A) vs the working-tree build (B)
N=${1:-3}
for i in $(seq $N); do
  echo -n "A "; FS_LIB=$PWD/paper_2411_15997_b200/lib/libfairserve_ab.so python bench.py --workload c4 --gen gpu --no-cpu-baseline --steps 10 --warmup 3 | python -c 'import json,sys; print(json.loads(sys.stdin.readline())["ms_per_step"])'
  echo -n "B "; python bench.py --workload c4 --gen gpu --no-cpu-baseline --steps 10 --warmup 3 | python -c 'import json,sys; print(json.loads(sys.stdin.readline())["ms_per_step"])'
done
