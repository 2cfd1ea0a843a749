# quick: profile parity subset + C4/C3 timings
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "profile or example_P" > gpurun_out/prof_tests.log 2>&1; echo "exit $?" >> gpurun_out/prof_tests.log
timeout 300 python tools/time_profile.py c4 5 > gpurun_out/time_c4.log 2>&1
tail -n 3 gpurun_out/prof_tests.log; cat gpurun_out/time_c4.log
