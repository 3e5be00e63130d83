TAG=${1:-k10}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_${TAG}.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_comb.py -q -x 2>&1 | tail -2
CMD="python bench.py --comb massive_12w --comb-kernel tc --steps 10 --warmup 3 --e2e-steps 3"
ncu --set full --clock-control none --cache-control none --import-source on -k regex:k10_ls -s 3 -c 1 -f -o gpurun_out/prof_${TAG}_ls $CMD > gpurun_out/ncu_${TAG}_ls.log 2>&1; echo "full ls rc $?"
ncu --set full --clock-control none --cache-control none --import-source on -k regex:k10_comb_tc -s 3 -c 1 -f -o gpurun_out/prof_${TAG}_main $CMD > gpurun_out/ncu_${TAG}_main.log 2>&1; echo "full main rc $?"
