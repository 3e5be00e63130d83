mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_comb.py -q -x 2>&1 | tail -1
for v in 2 1; do
CE_K10_LS=$v timeout 300 python bench.py --comb massive_12w --steps 50 --warmup 5 > gpurun_out/ls$v.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/ls$v.json').read().strip().splitlines()[-1]); print('ls$v', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))"
CE_K10_LS=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -c 20 --csv --log-file gpurun_out/ls$v.csv python bench.py --comb massive_12w --steps 10 --warmup 3 --e2e-steps 3 > /dev/null 2>&1
python tools/launches.py gpurun_out/ls$v.csv 2
done
