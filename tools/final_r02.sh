#!/bin/bash
# round-2 check on one B200: full GPU suite, smoke, the default (C5) bench line, C4 and C3 lines,
# the --impl reference line
mkdir -p gpurun_out
T=${1:-r02z}
python paper_2411_15997_b200/build.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${T}_smoke.log
tail -2 gpurun_out/${T}_smoke.log
timeout 1200 python bench.py --timings > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err
head -c 400 gpurun_out/${T}_bench_c5.json; echo
timeout 900 python bench.py --workload c4 --gen gpu --timings > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
head -c 400 gpurun_out/${T}_bench_c4.json; echo
timeout 1200 python bench.py --workload c3 --steps 2 --warmup 1 --timings > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
head -c 400 gpurun_out/${T}_bench_c3.json; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
head -c 400 gpurun_out/${T}_bench_ref.json; echo
