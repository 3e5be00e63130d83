mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1 || exit 1
for ck in 4096 2048 8192 16384; do for st in 20 100; do
CE_HOST_CHUNK_KB=$ck timeout 300 python bench.py --steps $st --warmup 5 --e2e-steps $st --sweep "" --no-cpu-baseline > gpurun_out/e2e_$ck_$st.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/e2e_$ck_$st.json').read().strip().splitlines()[-1]); e=d['e2e']; print('chunk $ck KB steps $st', '%.3g'%e['value'], '%.3g'%e.get('synchronous_call_value',0))"
done; done
python tools/pcie_bw.py
