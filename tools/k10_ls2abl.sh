mkdir -p gpurun_out
CMD="python bench.py --comb massive_12w --steps 10 --warmup 3 --e2e-steps 3"
for v in "nostore:-DK10_ABL_LS2_NOSTORE" "noload:-DK10_ABL_LS2_NOLOAD" "base:"; do
  name=${v%%:*}; flags=${v#*:}
  CE_NVCC_EXTRA="$flags" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > /dev/null 2>&1 || { echo "build failed"; continue; }
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none --cache-control none -k regex:k10_ls2 -c 2 --csv --log-file gpurun_out/ls2a.csv $CMD > /dev/null 2>&1
  echo "== $name"; python tools/launches.py gpurun_out/ls2a.csv 1
done
