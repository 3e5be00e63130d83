#!/bin/bash
# K4 pair mode build-flag matrix (same box): tools/pair_abl.sh  (PAIR_FLAGS="f1|f2|..." PAIR_CFGS=3,4,5)
mkdir -p gpurun_out
: > gpurun_out/pair_abl.log
IFS='|' read -ra FL <<< "${PAIR_FLAGS:-|-DK4_S_AB_P=4|-DK4_EPI_DB_P=1|-DK4_S_AB_P=4 -DK4_EPI_DB_P=1|-DK4_S_AB_P=2 -DK4_EPI_DB_P=1}"
for fl in "${FL[@]}"; do
  CE_NVCC_EXTRA="$fl" python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_pair.log 2>&1 || { echo "BUILD FAILED $fl" >> gpurun_out/pair_abl.log; continue; }
  echo "== flags: $fl" >> gpurun_out/pair_abl.log
  for pr in ${PAIR_MODES:-0 1}; do CE_K4_PAIR=$pr timeout 600 python tools/time_configs.py 3 ${PAIR_CFGS:-3,4,5} >> gpurun_out/pair_abl.log 2>&1; done
done
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build_pair.log 2>&1
cat gpurun_out/pair_abl.log
