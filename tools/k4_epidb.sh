mkdir -p gpurun_out
for v in "db1:-DK4_EPI_DB=1" "db0:"; do
  name=${v%%:*}; flags=${v#*:}
  CE_NVCC_EXTRA="$flags" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > /dev/null 2>&1 || { echo "build $name failed"; continue; }
  for c in 4 5 3; do
    timeout 300 python bench.py --config $c --steps 40 --warmup 5 --sweep "" --no-cpu-baseline > gpurun_out/db_$name_$c.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/db_$name_$c.json').read().strip().splitlines()[-1]); print('$name config $c', round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
