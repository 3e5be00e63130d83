mkdir -p gpurun_out
for v in "e16:-DK10_EPI_W=16" "e8:"; do
  name=${v%%:*}; flags=${v#*:}
  CE_NVCC_EXTRA="$flags" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > /dev/null 2>&1 || { echo "build $name failed"; continue; }
  timeout 900 python -m pytest tests/test_gpu_comb.py -q -x 2>&1 | tail -1
  timeout 300 python bench.py --comb massive_12w --steps 50 --warmup 5 > gpurun_out/comb_$name.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/comb_$name.json').read().strip().splitlines()[-1]); print('$name', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))"
done
