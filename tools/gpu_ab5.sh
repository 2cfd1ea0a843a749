#!/bin/bash
# compact head entries: parity, then sweep A/B (A = HEAD lib) incl. smaller carveouts, replay check
mkdir -p gpurun_out
T=${1:-hent}
python paper_2411_15997_b200/build.py > /dev/null
timeout 1200 python -m pytest tests -m gpu -x -q -k "sweep" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
AB=$PWD/paper_2411_15997_b200/lib/libfairserve_ab.so
for i in 1 2 3 4; do
  echo A; FS_LIB=$AB timeout 300 python tools/prof_sweep.py 4096
  echo B; timeout 300 python tools/prof_sweep.py 4096
done > gpurun_out/${T}_ab.log 2>&1
echo A >> gpurun_out/${T}_ab.log; FS_LIB=$AB timeout 300 python tools/prof_replay.py c2 >> gpurun_out/${T}_ab.log 2>&1
echo B >> gpurun_out/${T}_ab.log; timeout 300 python tools/prof_replay.py c2 >> gpurun_out/${T}_ab.log 2>&1
grep -v '^$' gpurun_out/${T}_ab.log | cut -c1-90
