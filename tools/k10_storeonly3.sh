mkdir -p gpurun_out
CMD="python bench.py --comb massive_12w --steps 10 --warmup 3 --e2e-steps 3"
for v in "so_v2:-DK10_ABL_STOREONLY" "so_v2_h3:-DK10_ABL_STOREONLY"; do
  name=${v%%:*}; flags=${v#*:}
  CE_NVCC_EXTRA="$flags" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > /dev/null 2>&1 || { echo "build failed"; exit 1; }
  CE_K10_L2HINT=1 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:k10_comb -c 2 --csv --log-file gpurun_out/so3.csv $CMD > /dev/null 2>&1
  echo "== $name"; python tools/launches.py gpurun_out/so3.csv 1
done
python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)'
