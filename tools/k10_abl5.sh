CMD="python bench.py --comb massive_12w --comb-kernel tc --steps 10 --warmup 3 --e2e-steps 3"
run() {
  CE_NVCC_EXTRA="$2" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > gpurun_out/build_abl_$1.log 2>&1 || { echo "build $1 failed"; tail -3 gpurun_out/build_abl_$1.log; return; }
  ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --cache-control none -k regex:k10_comb -c 3 --csv --log-file gpurun_out/abl5_$1.csv $CMD > /dev/null 2>&1
  echo "== $1"; python tools/launches.py gpurun_out/abl5_$1.csv 1
}
run noepi "-DK10_ABL_NOEPI"

run noepi_3commit "-DK10_ABL_NOEPI -DK10_ONE_COMMIT=0"
run base ""
python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)'
