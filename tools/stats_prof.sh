TAG=${1:-st}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1 || exit 1
for c in 4 5; do
CMD="python bench.py --stats --config $c --steps 3 --warmup 3"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --cache-control none -c 30 --csv --log-file gpurun_out/launches_${TAG}_c$c.csv $CMD > /dev/null 2>&1
echo "== config $c"; python tools/launches.py gpurun_out/launches_${TAG}_c$c.csv 6
done
ncu --set full --clock-control none --import-source on -k regex:k9_spectrum -s 2 -c 1 -f -o gpurun_out/prof_${TAG}_k9 python bench.py --stats --config 4 --steps 3 --warmup 3 > /dev/null 2>&1; echo "full k9 rc $?"
