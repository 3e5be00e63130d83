mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_stats.py -q -x 2>&1 | tail -3
for c in 4 5; do for pf in 1 0; do
CE_K9_PF=$pf timeout 300 python bench.py --stats --config $c --steps 20 --warmup 3 > gpurun_out/stats_pf${pf}_c$c.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/stats_pf${pf}_c$c.json').read().strip().splitlines()[-1]); print('config $c pf $pf', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
