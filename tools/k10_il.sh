mkdir -p gpurun_out
for v in "il_sa4:-DK10_INTERLEAVE=1 -DK10_SA_SLOTS=4" "il_sa2:-DK10_INTERLEAVE=1" "il_sa4_e16:-DK10_INTERLEAVE=1 -DK10_SA_SLOTS=4 -DK10_EPI_W=16" "base:"; do
  name=${v%%:*}; flags=${v#*:}
  CE_NVCC_EXTRA="$flags" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > gpurun_out/b_$name.log 2>&1 || { echo "build $name failed"; tail -3 gpurun_out/b_$name.log; continue; }
  timeout 600 python -m pytest tests/test_gpu_comb.py -q -x 2>&1 | tail -1
  for hint in 3 1; do
  CE_K10_L2HINT=$hint timeout 300 python bench.py --comb massive_12w --steps 50 --warmup 5 > gpurun_out/il_$name.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/il_$name.json').read().strip().splitlines()[-1]); print('$name hint $hint', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))"
  done
done
python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)'
