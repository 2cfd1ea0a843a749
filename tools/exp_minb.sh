for m in 1 4 5 6 7 8; do echo "MINB=$m"; FS_SWEEP_MINB=$m python tools/prof_sweep.py 4096; done 2>&1 | tee gpurun_out/minb.log
