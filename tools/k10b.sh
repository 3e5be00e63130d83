TAG=${1:-k10b}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_${TAG}.log 2>&1 || { tail -30 gpurun_out/build_${TAG}.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_comb.py -q -x 2>&1 | tail -5
for k in tc; do timeout 300 python bench.py --comb massive_12w --comb-kernel $k --steps 50 --warmup 5 > gpurun_out/comb_${TAG}_$k.json 2> gpurun_out/comb_${TAG}_$k.err; echo "bench $k rc $?"; tail -3 gpurun_out/comb_${TAG}_$k.err; done
for v in ; do CE_K10_L2HINT=$v timeout 300 python bench.py --comb massive_12w --comb-kernel tc --steps 50 --warmup 5 > gpurun_out/comb_${TAG}_hint$v.json 2>/dev/null; done
CE_K10_TMA_STORE=0 timeout 300 python bench.py --comb massive_12w --comb-kernel tc --steps 50 --warmup 5 > gpurun_out/comb_${TAG}_nost.json 2>/dev/null
python - <<PY
import json
for k in ("tc","hint0","nost"):
    try:
        d=json.loads(open(f"gpurun_out/comb_${TAG}_{k}.json").read().strip().splitlines()[-1])
        print(k, round(d["ms_per_step"]*1e3,1), "us", round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e: print(k, e)
PY
CMD="python bench.py --comb massive_12w --comb-kernel tc --steps 10 --warmup 3 --e2e-steps 3"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -c 40 --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > /dev/null 2>&1; echo "launch list rc $?"
