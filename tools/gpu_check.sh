# full GPU suite (minus the full-grid C5 test unless its golden exists) + C4/C3 profile timings
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
SEL=""
[ -f tests/golden/full_c5.json ] || SEL="--deselect tests/test_gpu_fullsize.py::test_sweep_c5_full"
timeout 1500 python -m pytest tests -m gpu -x -q $SEL > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/time_profile.py c4 5 > gpurun_out/time_c4.log 2>&1
timeout 300 python tools/time_profile.py c3 5 > gpurun_out/time_c3.log 2>&1
tail -n 4 gpurun_out/pytest_gpu.log; head -14 gpurun_out/time_c4.log; head -8 gpurun_out/time_c3.log
