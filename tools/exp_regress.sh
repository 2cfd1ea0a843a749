#!/bin/bash
python paper_2411_15997_b200/build.py > /dev/null
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr -Xptxas -O3 -o ab_old/libfairserve.so ab_old/pkg/csrc/fairserve.cu
timeout 1200 python tools/exp_regress.py ${ROUNDS:-3} 2>&1 | tee gpurun_out/exp_regress.log
timeout 300 python tools/time_step.py 3000 2>&1 | tail -2 | tee gpurun_out/time_step.log
