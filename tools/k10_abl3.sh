# K10 main-kernel ablations + L2 policy variants (whole-step bench times, launch lists)
CMD="python bench.py --comb massive_12w --comb-kernel tc --steps 10 --warmup 3 --e2e-steps 3"
run() {  # name flags env
  CE_NVCC_EXTRA="$2" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > gpurun_out/build_abl_$1.log 2>&1 || { echo "build $1 failed"; return; }
  env $3 python bench.py --comb massive_12w --comb-kernel tc --steps 50 --warmup 5 > gpurun_out/abl3_$1.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/abl3_$1.json').read().strip().splitlines()[-1]); print('$1', round(d['ms_per_step']*1e3,1), 'us', round(d['roofline']['frac'],3))"
  env $3 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -c 8 --csv --log-file gpurun_out/abl3_$1.csv $CMD > /dev/null 2>&1
  python tools/launches.py gpurun_out/abl3_$1.csv 2
}
run hint1 "" CE_K10_L2HINT=1
run hint3 "" CE_K10_L2HINT=3
run hint2 "" CE_K10_L2HINT=2
run hint0 "" CE_K10_L2HINT=0
run nostore "-DK10_ABL_NOSTORE" CE_K10_L2HINT=1
run noload "-DK10_ABL_NOLOAD" CE_K10_L2HINT=1
python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)'
