mkdir -p gpurun_out
for v in "c1:-DK10_CHUNK=1" "c2:-DK10_CHUNK=2" "c3:-DK10_CHUNK=3" "c4:-DK10_CHUNK=4" "c6:-DK10_CHUNK=6"; do
  name=${v%%:*}; flags=${v#*:}
  CE_NVCC_EXTRA="$flags" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > gpurun_out/b_$name.log 2>&1 || { echo "build $name failed"; tail -3 gpurun_out/b_$name.log; continue; }
  timeout 600 python -m pytest tests/test_gpu_comb.py -q -x 2>&1 | tail -1
  timeout 300 python bench.py --comb massive_12w --steps 50 --warmup 5 > gpurun_out/ch_$name.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ch_$name.json').read().strip().splitlines()[-1]); print('$name', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))"
done
python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)'
