#!/bin/bash
# K4 power mode (the statistics noise window) on CTA pairs: parity with pairs forced, then bench --stats A/B
mkdir -p gpurun_out
CE_K4_PAIR=1 timeout 900 python -m pytest tests/test_gpu_stats.py -x -q -m gpu > gpurun_out/pair_power_pytest.log 2>&1; echo "stats pytest (pairs forced) rc $?"; tail -2 gpurun_out/pair_power_pytest.log
for rep in 1 2; do for pr in 0 1; do for c in 4 5; do
  CE_K4_PAIR=$pr timeout 300 python bench.py --stats --config $c --steps 20 --warmup 3 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pair=$pr config $c: %.1f us' % (d['ms_per_step']*1e3))"
done; done; done 2>&1 | tee gpurun_out/pair_power.log
