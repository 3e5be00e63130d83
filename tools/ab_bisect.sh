#!/bin/bash
# Which single source change moves K4 out of its fast code-generation state?  Builds libce with each variant of
# K4's source (tools/ab_variants.py) in turn and times configs 3-4 on the same box; K4's own file is restored at the end.
# AB_VARIANTS="base v2_gfirst ..." AB_CFGS=3,4,5 tools/ab_bisect.sh
mkdir -p gpurun_out /tmp/k4cur
C=paper_1802_05427_b200/csrc
python tools/ab_variants.py > /dev/null || exit 1
cp $C/k4_block_lmmse_bf16x3.cu /tmp/k4cur/
: > gpurun_out/ab_bisect.log
for v in ${AB_VARIANTS:-base v1_template v2_gfirst v3_decode v4_bars v6_gridparam v8_gfirst_param v9_sraw v10_nks v12_srstep base}; do
  if [ $v = base ]; then cp /tmp/k4cur/k4_block_lmmse_bf16x3.cu $C/; else cp tools/ab_variants/$v.cu $C/k4_block_lmmse_bf16x3.cu; fi
  python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_ab.log 2>&1 || { echo "BUILD FAILED $v" >> gpurun_out/ab_bisect.log; continue; }
  echo "== $v (UIADD3 in k4_bf16x3: $(cuobjdump -sass paper_1802_05427_b200/_lib/libce.so | awk '/Function : .*k4_bf16x3E/{f=1;next} /Function :/{f=0} f' | grep -c UIADD3))" >> gpurun_out/ab_bisect.log
  CE_K4_PAIR=0 timeout 600 python tools/time_configs.py 3 ${AB_CFGS:-3,4} >> gpurun_out/ab_bisect.log 2>&1
done
cp /tmp/k4cur/k4_block_lmmse_bf16x3.cu $C/
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_ab.log 2>&1
cat gpurun_out/ab_bisect.log
