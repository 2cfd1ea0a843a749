python paper_2411_15997_b200/build.py > /dev/null
timeout 600 ncu --section WarpStateStats --section SourceCounters --import-source on --clock-control none -k regex:'^k_sweep' -c 1 -o gpurun_out/r01g_sweep python tools/prof_sweep.py 1184 50000 1000 > gpurun_out/r01g_sweep.log 2>&1
