mkdir -p gpurun_out
CMD="python bench.py --comb massive_12w --steps 10 --warmup 3 --e2e-steps 3"
for v in "so_lsu16:-DK10_ABL_STOREONLY -DK10_EPI_W=16 -DK10_ST_LSU" "lsu16:-DK10_EPI_W=16 -DK10_ST_LSU" "lsu8:-DK10_ST_LSU"; do
  name=${v%%:*}; flags=${v#*:}
  CE_NVCC_EXTRA="$flags" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > gpurun_out/b_$name.log 2>&1 || { echo "build $name failed"; tail -3 gpurun_out/b_$name.log; continue; }
  CE_K10_L2HINT=1 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:k10_comb -c 2 --csv --log-file gpurun_out/lsu_$name.csv $CMD > /dev/null 2>&1
  echo "== $name"; python tools/launches.py gpurun_out/lsu_$name.csv 1
done
CE_NVCC_EXTRA="-DK10_EPI_W=16 -DK10_ST_LSU" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_comb.py -q -x 2>&1 | tail -1
python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)'
