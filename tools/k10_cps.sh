mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_comb.py -q -x 2>&1 | tail -3
for c in massive_12w paper_12w; do timeout 300 python bench.py --comb $c --steps 50 --warmup 5 > gpurun_out/comb_cps1_$c.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/comb_cps1_$c.json').read().strip().splitlines()[-1]); print('cps1 $c', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3), d['config']['kernel'])"; done
CE_NVCC_EXTRA="-DK10_CPS=2" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > /dev/null 2>&1 || { echo cps2 build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_comb.py -q -x 2>&1 | tail -2
timeout 300 python bench.py --comb massive_12w --steps 50 --warmup 5 > gpurun_out/comb_cps2.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/comb_cps2.json').read().strip().splitlines()[-1]); print('cps2', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))"
python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)'
