#!/bin/bash
# detail sections for the HBM-bound kernels on C3 (10M calls)
TAG=${1:-r01e}
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section LaunchStats \
  --section Occupancy --section SourceCounters --section ComputeWorkloadAnalysis --import-source on --clock-control none \
  -k regex:'k_prof_stream|k_win_scan|k_act_flags|k_act_decide|k_radix_scatter|k_q_count' -c 8 \
  -o gpurun_out/${TAG}_hbm python tools/prof_stages.py c3 > gpurun_out/${TAG}_hbm.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches_c3.csv python tools/prof_stages.py c3 > /dev/null 2>&1
ls -la gpurun_out
