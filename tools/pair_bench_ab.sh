#!/bin/bash
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_pair.log 2>&1 || { echo BUILD FAILED; exit 1; }
for rep in 1 2; do for pr in 0 auto; do
  if [ $pr = auto ]; then unset CE_K4_PAIR; else export CE_K4_PAIR=$pr; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 --sweep-steps 20 > gpurun_out/bench_ab_${pr}_${rep}.json 2>/dev/null
  python - <<PY
import json
d=json.loads(open('gpurun_out/bench_ab_${pr}_${rep}.json').read().strip().splitlines()[-1])
print('pair=${pr} rep=${rep} c3 %.2f us' % (d['ms_per_step']*1e3), ' '.join('%s %.1f us (%.3f) %s MHz' % (s['workload'][:7], s['ms_per_step']*1e3, s['roofline']['frac'], s['clocks']['sm_mhz']) for s in d['sweep']))
PY
done; done
