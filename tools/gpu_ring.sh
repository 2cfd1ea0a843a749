#!/bin/bash
# sweep ring-capacity A/B (interleaved) + validation fast path C4 timing
mkdir -p gpurun_out
python paper_2411_15997_b200/build.py > /dev/null
for c in 512 128 512 128 64 256; do FS_SWEEP_RING_CAP=$c timeout 300 python tools/exp_ring.py 2>&1 | tail -2; done > gpurun_out/ring.log
cat gpurun_out/ring.log
