"""Brief ncu summary: duration, issue, pipes, smem wavefronts/conflicts, L2, stall reasons."""
import csv, subprocess, sys
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
def g(k):
    return d.get(k, "?")
keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_bytes.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum"]
for k in keys:
    print(f"{k:70s} {g(k)}")
st = sorted(((k, float(x.replace(',', '') or 0)) for k, x in d.items()
             if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")), key=lambda kv: -kv[1])
tot = sum(x for _, x in st)
for k, x in st[:12]:
    print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {x / tot * 100:5.1f}%")
