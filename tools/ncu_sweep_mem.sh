#!/bin/bash
# memory/stall sections of k_sweep at full size (no SASS instrumentation: finishes in minutes)
TAG=${1:-r01d}; S=${2:-1184}
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
timeout 900 ncu --section LaunchStats --section Occupancy --section WarpStateStats --section SchedulerStats \
  --section MemoryWorkloadAnalysis --section MemoryWorkloadAnalysis_Tables --section ComputeWorkloadAnalysis \
  --metrics smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct \
  --clock-control none -k regex:'^k_sweep' -c 1 -o gpurun_out/${TAG}_sweep python tools/prof_sweep.py $S > gpurun_out/${TAG}_sweep.log 2>&1
ls -la gpurun_out
