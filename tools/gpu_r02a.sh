# round 2 first check on one B200: GPU suite (minus the full-grid C5 test until its golden exists), smoke, default bench
mkdir -p gpurun_out
nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_fullsize.py::test_sweep_c5_full > gpurun_out/pytest_r02a.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r02a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02a.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_r02a.log
timeout 1200 python bench.py --timings > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo "bench exit $?" >> gpurun_out/bench_r02a.err
tail -3 gpurun_out/pytest_r02a.log; tail -2 gpurun_out/smoke_r02a.log; cat gpurun_out/bench_r02a.json | head -c 3000
