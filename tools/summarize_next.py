"""Key ncu --set full counters of the NEXT-row kernels (statistics K8 / K7c / K7a, comb-pilot K6) into
profiles/ncu_next_TAG.json.

usage: python tools/summarize_next.py TAG   (reads gpurun_out/next_{k8,k7c,k7a,k6}_TAG.ncu-rep; see tools/profile_next.sh)
"""
import csv
import io
import json
import os
import subprocess
import sys

TAG = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
        "launch__shared_mem_per_block_dynamic"]
WHAT = {"k8": "k8_gram, statistics config 4 (lags on tcgen05)",
        "k7c": "k7_noise, statistics config 4 (streamed FFMA2 noise window)",
        "k7a": "k7_accumulate, statistics config 3 (lags + noise window, FP32)",
        "k6": "k6_estimate_g<12W>, comb massive_12w"}


def full(p):
    txt = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {k: {"value": v[h.index(k)], "unit": u[h.index(k)]} for k in KEYS if k in h}
    stalls = [(k, float(v[h.index(k)].replace(",", "") or 0)) for k in h
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    tot = sum(x for _, x in stalls) or 1
    d["top_stalls_pct"] = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(100 * x / tot, 1)
                           for k, x in sorted(stalls, key=lambda z: -z[1])[:6]}
    return d


out = {"tag": TAG, "kernels": {}}
for key, what in WHAT.items():
    p = os.path.join(G, f"next_{key}_{TAG}.ncu-rep")
    if os.path.exists(p):
        out["kernels"][key] = {"what": what, "counters": full(p)}
json.dump(out, open(os.path.join(ROOT, "profiles", f"ncu_next_{TAG}.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
