#!/bin/bash
# K4 pair mode: resident-cluster count and grid-size sweep (same box)
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_pair.log 2>&1 || { echo BUILD FAILED; tail -20 gpurun_out/build_pair.log; exit 1; }
{
CE_K4_PAIR=0 timeout 600 python tools/time_configs.py 3 3,4,5
CE_K4_DEBUG=1 CE_K4_PAIR=1 timeout 600 python tools/time_configs.py 3 3,4,5
for n in ${PAIR_SWEEP:-72 70 66 64 60 56}; do CE_K4_PAIR=1 CE_K4_PAIRS=$n timeout 600 python tools/time_configs.py 3 3,4,5; done
} > gpurun_out/pair_sweep.log 2>&1
cat gpurun_out/pair_sweep.log
