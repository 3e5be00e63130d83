"""Summarise ncu outputs into profiles/: launch-list shares and --set full key counters (JSON + text).

usage: python tools/summarize_ncu.py TAG  (reads gpurun_out/launches_TAG.csv, prof_c3_TAG / prof_c5_TAG .ncu-rep)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

TAG = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")
G = os.path.join(ROOT, "gpurun_out")


def short(name):
    for k in ("k4_bf16x3", "k5_pair", "k3_tf32x3", "k2_simt", "k1_levinson", "k1_schur", "k1_refine", "k1_trench", "k1_mirror", "k3_build_bank",
              "k4_build_bank"):
        if k in name:
            return k
    return name[:40]


def launches():
    rows = list(csv.reader(open(os.path.join(G, f"launches_{TAG}.csv"))))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    per = defaultdict(list)
    for r in rows[start + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", ""))
            unit = d["Metric Unit"]
            v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
            per[short(d["Kernel Name"])].append(v)
    tot = sum(sum(v) for v in per.values())
    return {k: {"launches": len(v), "avg_us": sum(v) / len(v), "share": sum(v) / tot} for k, v in per.items()}


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
        "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_l1tex2xbar_write_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "launch__shared_mem_per_block_dynamic"]


def full(rep):
    p = os.path.join(G, rep + ".ncu-rep")
    if not os.path.exists(p):
        return None
    txt = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            d[k] = {"value": v[i], "unit": u[i]}
    stalls = [(k, float(v[h.index(k)].replace(",", "") or 0)) for k in h
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    tot = sum(x for _, x in stalls) or 1
    d["top_stalls_pct"] = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(100 * x / tot, 1)
                           for k, x in sorted(stalls, key=lambda z: -z[1])[:6]}
    return d


def to_bytes(e):
    val = float(e["value"].replace(",", ""))
    return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(e["unit"], 1)


summ = {"tag": TAG, "launch_list": launches(), "kernels": {}}
for rep, cfg in ((f"prof_c3_{TAG}", "config3"), (f"prof_c5_{TAG}", "config5")):
    f = full(rep)
    if f is None:
        continue
    entry = {"config": cfg, "counters": f}
    if "dram__bytes_read.sum" in f:
        entry["dram_bytes_per_launch"] = to_bytes(f["dram__bytes_read.sum"]) + to_bytes(f["dram__bytes_write.sum"])
    summ["kernels"]["k4_bf16x3" + ("" if cfg == "config3" else "_config5")] = entry
os.makedirs(OUT, exist_ok=True)
json.dump(summ, open(os.path.join(OUT, f"ncu_summary_{TAG}.json"), "w"), indent=1)
json.dump(summ, open(os.path.join(OUT, "ncu_summary.json"), "w"), indent=1)
print(json.dumps(summ, indent=1))
