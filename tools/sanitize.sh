#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every C-ABI call (tools/sanitize_run.py:
# C1 and a 100k-call C2-shaped trace); summaries in gpurun_out/sanitizer_<tool>.log
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
for tool in memcheck synccheck racecheck; do
  arg=""
  [ "$tool" = "racecheck" ] && arg="small"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py $arg \
    > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitizer_$tool.log
  tail -3 gpurun_out/sanitizer_$tool.log
done
