#!/bin/bash
# ncu evidence for round 2 (one GPU, under gpurun):
#   <tag>_launches.csv   every launch of one default bench step (gpu__time_duration, cold/serialised)
#   <tag>_sweep.csv      k_sweep over the bench's 4096 C5 scenarios: instructions, duration, dram bytes, hit rates
#   <tag>_replay.csv     k_replay_warp (the C2 single replay): instructions, cycles, duration, dram bytes
#   <tag>_c4_dram.csv    every kernel of one C4 profile build (100M calls): duration, dram bytes
#   <tag>_c3_act_dram.csv every kernel of the C3 ACT calls (tools/time_act.py): duration, dram bytes
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
M2="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 0 > gpurun_out/${TAG}_launches_bench.log 2>&1
timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:'^k_sweep' --csv --log-file gpurun_out/${TAG}_sweep.csv \
    python tools/prof_sweep.py 4096 > gpurun_out/${TAG}_sweep.log 2>&1
echo '"0","0","x","x","k_sweep","1","7","(1,1,1)","(1,1,1)","0","10.0","info","scenarios","","4096"' >> gpurun_out/${TAG}_sweep.csv
timeout 600 ncu --metrics smsp__inst_executed.sum,sm__cycles_elapsed.max,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:'^k_replay_warp' --csv --log-file gpurun_out/${TAG}_replay.csv \
    python tools/prof_replay.py c2 0 1 > gpurun_out/${TAG}_replay.log 2>&1
timeout 900 ncu --metrics $M2 --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/${TAG}_c4_dram.csv \
    python tools/time_profile.py c4 1 > gpurun_out/${TAG}_c4_dram.log 2>&1
timeout 900 ncu --metrics $M2 --clock-control none -k regex:'^k_' --csv --log-file gpurun_out/${TAG}_c3_act_dram.csv \
    python tools/time_act.py c3 1 always > gpurun_out/${TAG}_c3_act_dram.log 2>&1
ls -la gpurun_out/${TAG}_*
