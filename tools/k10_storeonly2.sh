mkdir -p gpurun_out
CMD="python bench.py --comb massive_12w --steps 10 --warmup 3 --e2e-steps 3"
CE_NVCC_EXTRA="-DK10_ABL_STOREONLY -DK10_EPI_W=16" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > /dev/null 2>&1 || { echo "build failed"; exit 1; }
for e in "CE_K10_L2HINT=3" "CE_K10_L2HINT=1" "CE_K10_L2HINT=0" "CE_K10_TMA_STORE=0"; do
  env $e ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:k10_comb -c 2 --csv --log-file gpurun_out/so2.csv $CMD > /dev/null 2>&1
  echo "== $e"; python tools/launches.py gpurun_out/so2.csv 1
done
python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)'
