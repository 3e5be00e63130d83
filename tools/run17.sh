timeout 900 python -m pytest tests/test_gpu_comb.py -x -q > gpurun_out/pytest_comb.txt 2>&1; echo "pytest comb rc $?"; tail -15 gpurun_out/pytest_comb.txt
for c in massive_12w paper_12w paper_3w; do
timeout 300 python bench.py --comb $c --steps 200 --warmup 10 > gpurun_out/bench_comb_$c.json 2> gpurun_out/bench_comb_$c.err; echo "bench $c rc $?"; cat gpurun_out/bench_comb_$c.json | cut -c1-600; tail -2 gpurun_out/bench_comb_$c.err
done
