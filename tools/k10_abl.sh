# k10_ls ablations: launch lists of variants built with CE_NVCC_EXTRA
CMD="python bench.py --comb massive_12w --comb-kernel tc --steps 10 --warmup 3 --e2e-steps 3"
for v in "base:" "nostore:-DK10_ABL_LS_NOSTORE" "noload:-DK10_ABL_LS_NOLOAD" "rows1:-DK10_LSR_ROWS=1" "rows2:-DK10_LSR_ROWS=2" "rows8:-DK10_LSR_ROWS=8"; do
  name=${v%%:*}; flags=${v#*:}
  CE_NVCC_EXTRA="$flags" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > gpurun_out/build_abl_$name.log 2>&1 || { echo "build $name failed"; continue; }
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum --clock-control none --cache-control none -k regex:k10_ls -c 6 --csv --log-file gpurun_out/abl_$name.csv $CMD > /dev/null 2>&1
  echo "== $name"; python tools/launches.py gpurun_out/abl_$name.csv 2
done
python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)'
