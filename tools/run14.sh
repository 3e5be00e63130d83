timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_v14.txt 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_v14.txt
timeout 600 python bench.py > gpurun_out/bench_v14.json 2> gpurun_out/bench_v14.err; echo "bench rc $?"; cat gpurun_out/bench_v14.json
bash tools/sweep.sh "0 4" "3 4 5" 200
