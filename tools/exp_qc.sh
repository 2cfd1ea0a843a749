#!/bin/bash
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fullsize.py -q -x -k "profile" 2>&1 | tail -2
for cfg in "12288 256" "28672 2048" "28672 256" "4096 64"; do set -- $cfg; echo "PRIV=$1 NSUB=$2"; FS_QC_PRIV=$1 FS_QC_NSUB=$2 timeout 300 python tools/time_profile.py c4 5 | grep -E "profile|q_"; done 2>&1 | tee gpurun_out/exp_qc.log
