# K10 profile: launch list (per-kernel times) + ncu --set full of k10_comb_tc and k10_ls on massive_12w
mkdir -p gpurun_out
TAG=${1:-k10}
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_${TAG}.log 2>&1 || exit 1
CMD="python bench.py --comb massive_12w --comb-kernel tc --steps 10 --warmup 3 --e2e-steps 3"
eval $CMD > gpurun_out/plain_${TAG}.json 2>&1 || { tail gpurun_out/plain_${TAG}.json; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > /dev/null 2>&1; echo "launch list rc $?"
ncu --set full --clock-control none --import-source on -k regex:k10_comb_tc -s 3 -c 1 -f -o gpurun_out/prof_${TAG}_main $CMD > gpurun_out/ncu_${TAG}_main.log 2>&1; echo "full main rc $?"
ncu --set full --clock-control none --import-source on -k regex:k10_ls -s 3 -c 1 -f -o gpurun_out/prof_${TAG}_ls $CMD > gpurun_out/ncu_${TAG}_ls.log 2>&1; echo "full ls rc $?"
