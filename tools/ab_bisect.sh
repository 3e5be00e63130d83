#!/bin/bash
# Which source change costs the single-CTA kernel 9 % on config 3?  Variants of K4's own source (tools/ab_old/variants).
mkdir -p gpurun_out /tmp/k4cur
C=paper_1802_05427_b200/csrc
cp $C/k4_block_lmmse_bf16x3.cu /tmp/k4cur/
: > gpurun_out/ab_bisect.log
for v in ${AB_VARIANTS:-base v1_template v2_gfirst v3_decode v4_bars base}; do
  if [ $v = base ]; then cp /tmp/k4cur/k4_block_lmmse_bf16x3.cu $C/; else cp tools/ab_old/variants/$v.cu $C/k4_block_lmmse_bf16x3.cu; fi
  python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_ab.log 2>&1 || { echo "BUILD FAILED $v" >> gpurun_out/ab_bisect.log; continue; }
  echo "== $v" >> gpurun_out/ab_bisect.log
  CE_K4_PAIR=0 timeout 600 python tools/time_configs.py 3 3,4 >> gpurun_out/ab_bisect.log 2>&1
done
cp /tmp/k4cur/k4_block_lmmse_bf16x3.cu $C/
cat gpurun_out/ab_bisect.log
