#!/bin/bash
# ncu evidence for one round (run under gpurun on ONE GPU):
#   gpurun_out/<tag>_launches.csv   every launch of one default bench step (gpu__time_duration, cold/serialised)
#   gpurun_out/<tag>_sweep.csv      k_sweep over the bench's 4096 C5 scenarios: instructions, duration, dram bytes
#   gpurun_out/<tag>_replay.csv     k_replay on C2: instructions, cycles, duration, dram bytes
#   gpurun_out/<tag>_hbm.csv        the HBM-bound kernels on C3 (dram bytes, throughput, duration)
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_launches_bench.log 2>&1
ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct \
    --clock-control none -k regex:'^k_sweep' --csv --log-file gpurun_out/${TAG}_sweep.csv \
    python tools/prof_sweep.py 4096 > gpurun_out/${TAG}_sweep.log 2>&1
echo '"0","0","x","x","k_sweep","1","7","(1,1,1)","(1,1,1)","0","10.0","info","scenarios","","4096"' >> gpurun_out/${TAG}_sweep.csv
ncu --metrics smsp__inst_executed.sum,sm__cycles_elapsed.max,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:'^k_replay$' --csv --log-file gpurun_out/${TAG}_replay.csv \
    python tools/prof_replay.py c2 0 1 > gpurun_out/${TAG}_replay.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:'k_prof_stream|k_radix_scatter|k_win_scan|k_win_peaks|k_act_flags|k_act_decide|k_act_walk|k_q_count|k_pack_records|k_val_' \
    --csv --log-file gpurun_out/${TAG}_hbm.csv python tools/prof_stages.py c3 > gpurun_out/${TAG}_hbm.log 2>&1
echo done
