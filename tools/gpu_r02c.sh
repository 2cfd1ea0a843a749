bash tools/gpu_prof_quick.sh
timeout 300 python -m pytest tests/test_gpu_edge.py -x -q > gpurun_out/edge.log 2>&1; tail -n 2 gpurun_out/edge.log
SKIP=6 CNT=8 bash tools/ncu_prof_c4.sh r02c "k_os_pass|k_win_pieces|k_q_count|k_vf_|k_os_tile_hist"
