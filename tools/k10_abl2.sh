# K10 PDL ablations: whole-step time (bench) and per-kernel launch list
CMD="python bench.py --comb massive_12w --comb-kernel tc --steps 10 --warmup 3 --e2e-steps 3"
for v in "base:" "late:-DK10_LS_LATE_TRIGGER" "nopdl:-DK10_NO_PDL"; do
  name=${v%%:*}; flags=${v#*:}
  CE_NVCC_EXTRA="$flags" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > gpurun_out/build_abl_$name.log 2>&1 || { echo "build $name failed"; continue; }
  python bench.py --comb massive_12w --comb-kernel tc --steps 50 --warmup 5 > gpurun_out/abl2_$name.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/abl2_$name.json').read().strip().splitlines()[-1]); print('$name', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))"
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 8 --csv --log-file gpurun_out/abl2_$name.csv $CMD > /dev/null 2>&1
  python tools/launches.py gpurun_out/abl2_$name.csv 2
done
python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)'
