timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_v19.txt 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/pytest_v19.txt
bash tools/sweep.sh "0 1 2" "6" 100
bash tools/sweep.sh "0" "3" 1000
