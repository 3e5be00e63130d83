#!/bin/bash
# ncu evidence for the bench workload: launch list (cold, serialised) + one --set full capture of the hot kernel.
TAG=${1:-r01}
CMD="python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 3"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch list rc $?"
$CMD > gpurun_out/plain2_${TAG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k4_bf16x3 -s 10 -c 1 -f -o gpurun_out/prof_c3_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "full c3 rc $?"
CMD5="python bench.py --config 5 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 3"
$CMD5 > gpurun_out/plain5_${TAG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k4_bf16x3 -s 3 -c 1 -f -o gpurun_out/prof_c5_${TAG} $CMD5 > gpurun_out/ncu_full5_${TAG}.log 2>&1
echo "full c5 rc $?"
python -c "
import torch,time
x=torch.empty(14745600//4,dtype=torch.float32,device='cuda')
ys=[torch.empty_like(x) for _ in range(8)]; xs=[torch.empty_like(x) for _ in range(8)]
for i in range(20): ys[i%8].copy_(xs[i%8])
torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(1000): ys[i%8].copy_(xs[i%8])
e1.record(); torch.cuda.synchronize(); print('torch copy 14.7 MB back-to-back: %.2f us per copy' % (e0.elapsed_time(e1)))
" > gpurun_out/copy_c3_${TAG}.txt 2>&1; cat gpurun_out/copy_c3_${TAG}.txt
