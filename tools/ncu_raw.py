"""Summarise an ncu --page raw --csv export: stall reasons and key counters."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, units = rows[0], rows[1]
for v in rows[2:]:
    d = dict(zip(h, v))
    print("==", d.get("Kernel Name", "")[:80], "duration", d.get("gpu__time_duration.sum"))
    keys = [k for k in h if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")]
    vals = sorted(((float(d[k].replace(",", "")) if d[k] else 0, k) for k in keys), reverse=True)
    tot = sum(x for x, _ in vals) or 1
    for val, k in vals[:12]:
        print(f"  {100*val/tot:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_','')}")
    for k in sys.argv[2:] or ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.sum",
              "sm__inst_executed.sum", "smsp__inst_executed_op_shared_ld.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
              "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
              "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]:
        if k in h:
            print(f"  {k} = {d[k]} {units[h.index(k)]}")
