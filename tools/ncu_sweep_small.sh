#!/bin/bash
# stall reasons + source-level hot spots of k_sweep and k_replay on reduced traces (full-set on the
# 1M-call trace does not finish under ncu's SASS instrumentation)
TAG=${1:-r01c}; S=${2:-1184}; N=${3:-50000}
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
timeout 600 ncu --section LaunchStats --section Occupancy --section WarpStateStats --section SchedulerStats \
  --section MemoryWorkloadAnalysis --section SourceCounters --section ComputeWorkloadAnalysis --import-source on \
  --clock-control none -k regex:'^k_sweep' -c 1 -o gpurun_out/${TAG}_sweep python tools/prof_sweep.py $S $N 1000 > gpurun_out/${TAG}_sweep.log 2>&1
timeout 600 ncu --section LaunchStats --section WarpStateStats --section SchedulerStats --section SourceCounters \
  --section MemoryWorkloadAnalysis --import-source on \
  --clock-control none -k regex:'^k_replay$' -c 1 -o gpurun_out/${TAG}_replay python tools/prof_replay.py c2 $N 1 > gpurun_out/${TAG}_replay.log 2>&1
python tools/prof_sweep.py $S $N 1000 >> gpurun_out/${TAG}_sweep.log 2>&1
ls -la gpurun_out
