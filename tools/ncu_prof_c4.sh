# ncu --set full of the C4 profile's top kernels (one build, after the warm-up call), for the
# source-level stall picture.  Usage (under gpurun): bash tools/ncu_prof_c4.sh TAG [regex]
TAG=${1:-r02}
RX=${2:-'k_os_pass|k_win_pieces|k_prof_stream|k_q_count|k_val_links|k_val_range'}
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
ncu --set full --clock-control none --import-source on -k regex:"$RX" -s ${SKIP:-8} -c ${CNT:-7} \
    -o gpurun_out/${TAG}_c4 python tools/time_profile.py c4 1 > gpurun_out/${TAG}_c4_ncu.log 2>&1
ncu -i gpurun_out/${TAG}_c4.ncu-rep --page raw --csv > gpurun_out/${TAG}_c4_raw.csv 2>/dev/null
ls -la gpurun_out/${TAG}_c4*
