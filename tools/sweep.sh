#!/bin/bash
# Usage: tools/sweep.sh "<kernels>" "<configs>" [steps]   -- one bench line summary per (kernel, config)
K=${1:-"0"}; C=${2:-"3 4 5"}; S=${3:-300}
for k in $K; do for c in $C; do
  timeout 300 python bench.py --config $c --kernel $k --steps $S --warmup 20 --no-cpu-baseline --e2e-steps 3 > gpurun_out/sw_k${k}_c${c}.json 2> gpurun_out/sw_k${k}_c${c}.err
  python - "$k" "$c" <<'PY'
import json, sys
k, c = sys.argv[1], sys.argv[2]
try:
    d = json.load(open(f"gpurun_out/sw_k{k}_c{c}.json")); r = d["roofline"]
    print(f"k{k} c{c} {d['config']['kernel']:18s} {d['ms_per_step']*1e3:9.2f} us  {d['value']:.3e} est/s  {r['bound']} frac {r['frac']:.3f} hbm {r['hbm_frac']:.3f}  clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
except Exception as e:
    print(f"k{k} c{c} FAILED {e}; " + open(f"gpurun_out/sw_k{k}_c{c}.err").read()[-300:])
PY
done; done
