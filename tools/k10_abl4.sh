CMD="python bench.py --comb massive_12w --comb-kernel tc --steps 10 --warmup 3 --e2e-steps 3"
run() {  # name flags
  CE_NVCC_EXTRA="$2" python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)' > gpurun_out/build_abl_$1.log 2>&1 || { echo "build $1 failed"; tail -3 gpurun_out/build_abl_$1.log; return; }
  CE_K10_L2HINT=3 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k10_comb -c 4 --csv --log-file gpurun_out/abl4_$1.csv $CMD > /dev/null 2>&1
  echo "== $1"; python tools/launches.py gpurun_out/abl4_$1.csv 2
}
run ns_sa2_sb4 "-DK10_ABL_NOSTORE"
run ns_sa2_sb2 "-DK10_ABL_NOSTORE -DK10_SB_STAGES=2"
run ns_sa2_sb6 "-DK10_ABL_NOSTORE -DK10_SB_STAGES=6"
run ns_sa4_sb4 "-DK10_ABL_NOSTORE -DK10_SA_SLOTS=4"
run ns_sa6_sb4 "-DK10_ABL_NOSTORE -DK10_SA_SLOTS=6 -DK10_SB_STAGES=3"
run sa4_sb4 "-DK10_SA_SLOTS=4"
run sa6_sb3 "-DK10_SA_SLOTS=6 -DK10_SB_STAGES=3"
python -c 'import paper_1802_05427_b200.build as b; b.build(force=True)'
