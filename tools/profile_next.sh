#!/bin/bash
# ncu --set full captures of the NEXT-row kernels (one launch each, after the same command ran clean without ncu).
TAG=${1:-r01}
S4="python bench.py --stats --config 4 --steps 3 --warmup 3 --no-cpu-baseline"
S3="python bench.py --stats --config 3 --steps 3 --warmup 3 --no-cpu-baseline"
C12="python bench.py --comb massive_12w --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2"
for cmd in "$S4" "$S3" "$C12"; do timeout 300 $cmd > /dev/null 2>&1 || echo "plain run failed: $cmd"; done
cap() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 2 -c 1 -f -o gpurun_out/next_$1_${TAG} $3 > gpurun_out/ncu_next_$1_${TAG}.log 2>&1; echo "next $1 rc $?"; }
cap k8 k8_gram "$S4"
cap k7c k7_noise "$S4"
cap k7a k7_accumulate "$S3"
cap k6 k6_estimate_g "$C12"
