#!/bin/bash
# Same-box A/B of the K4 single-CTA path: the kernel file of commit 64a99ea (before the pair-mode template) vs HEAD
mkdir -p gpurun_out /tmp/k4new
C=paper_1802_05427_b200/csrc
cp $C/k4_block_lmmse_bf16x3.cu $C/tc_ptx.cuh /tmp/k4new/
: > gpurun_out/ab_old.log
for rep in 1 2; do
  cp tools/ab_old/k4_block_lmmse_bf16x3.cu.old $C/k4_block_lmmse_bf16x3.cu; cp tools/ab_old/tc_ptx.cuh.old $C/tc_ptx.cuh
  python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_ab.log 2>&1 || { echo "OLD BUILD FAILED"; tail gpurun_out/build_ab.log; }
  echo "== old (64a99ea)" >> gpurun_out/ab_old.log
  timeout 600 python tools/time_configs.py 3 3,4,5 >> gpurun_out/ab_old.log 2>&1
  timeout 300 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline --sweep "" --e2e-steps 3 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("bench2000 %.2f us direct %.2f" % (d["ms_per_step"]*1e3, d["direct_launch"]["ms_per_step"]*1e3))' >> gpurun_out/ab_old.log
  cp /tmp/k4new/k4_block_lmmse_bf16x3.cu /tmp/k4new/tc_ptx.cuh $C/
  python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_ab.log 2>&1 || { echo "NEW BUILD FAILED"; tail gpurun_out/build_ab.log; }
  echo "== new (HEAD)" >> gpurun_out/ab_old.log
  CE_K4_PAIR=0 timeout 600 python tools/time_configs.py 3 3,4,5 >> gpurun_out/ab_old.log 2>&1
  timeout 300 python bench.py --steps 2000 --warmup 50 --no-cpu-baseline --sweep "" --e2e-steps 3 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("bench2000 %.2f us direct %.2f" % (d["ms_per_step"]*1e3, d["direct_launch"]["ms_per_step"]*1e3))' >> gpurun_out/ab_old.log
done
cat gpurun_out/ab_old.log
