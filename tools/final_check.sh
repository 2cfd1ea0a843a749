# round-end check on one B200: full GPU suite, smoke, the default (C5) and C4 bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r01z.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r01z.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01z.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_r01z.log
timeout 900 python bench.py --timings > gpurun_out/bench_c5z.json 2> gpurun_out/bench_c5z.err
timeout 600 python bench.py --workload c4 --gen gpu --timings > gpurun_out/bench_c4z.json 2> gpurun_out/bench_c4z.err
tail -2 gpurun_out/pytest_r01z.log; tail -1 gpurun_out/smoke_r01z.log; head -c 300 gpurun_out/bench_c5z.json; echo; head -c 300 gpurun_out/bench_c4z.json
