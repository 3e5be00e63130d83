set -x
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_k10a.log 2>&1 || { tail -30 gpurun_out/build_k10a.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_comb.py -q -x 2>&1 | tail -25
for k in tc simt; do timeout 300 python bench.py --comb massive_12w --comb-kernel $k --steps 50 --warmup 5 > gpurun_out/comb_k10a_$k.json 2> gpurun_out/comb_k10a_$k.err; echo "bench $k rc $?"; tail -3 gpurun_out/comb_k10a_$k.err; done
python - <<'PY'
import json
for k in ("tc","simt"):
    try:
        d=json.loads(open(f"gpurun_out/comb_k10a_{k}.json").read().strip().splitlines()[-1])
        print(k, d["ms_per_step"]*1e3, "us", d["roofline"]["frac"], d["clocks"])
    except Exception as e: print(k, e)
PY
