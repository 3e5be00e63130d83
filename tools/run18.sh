CMD="python bench.py --comb massive_12w --steps 10 --warmup 3"
$CMD > gpurun_out/plain_comb.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k6_estimate -s 3 -c 1 -f -o gpurun_out/prof_comb $CMD > gpurun_out/ncu_comb.log 2>&1; echo "ncu rc $?"
