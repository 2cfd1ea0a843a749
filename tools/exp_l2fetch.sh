#!/bin/bash
# C4 step with the default L2 fetch granularity vs FS_L2_FETCH=$1
for i in 1 2; do
  echo -n "A "; python bench.py --workload c4 --gen gpu --no-cpu-baseline --steps 10 --warmup 3 --timings 2> /tmp/a.err | python -c 'import json,sys; print(json.loads(sys.stdin.readline())["ms_per_step"])'; grep -E "win_scan|radix_scatter|prof_stream" /tmp/a.err
  echo -n "B "; FS_L2_FETCH=$1 python bench.py --workload c4 --gen gpu --no-cpu-baseline --steps 10 --warmup 3 --timings 2> /tmp/b.err | python -c 'import json,sys; print(json.loads(sys.stdin.readline())["ms_per_step"])'; grep -E "win_scan|radix_scatter|prof_stream" /tmp/b.err
done
