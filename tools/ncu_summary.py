"""Extract the judged metrics of an ncu --set full capture into profiles/ (json + text)."""
import csv
import io
import json
import subprocess
import sys

rep, out_json = sys.argv[1], sys.argv[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, units = rows[0], rows[1]
res = []
for v in rows[2:]:
    d = dict(zip(h, v))
    rec = {"kernel": d.get("Kernel Name", "")[:120]}
    U = dict(zip(h, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
             "msecond": 1.0, "second": 1e3}
    for k in keys:
        if k in d:
            try:
                val = float(d[k].replace(",", ""))
            except ValueError:
                rec[k] = d[k]
                continue
            u = U.get(k, "")
            if u in scale:
                val *= scale[u]
                rec[k + " [" + ("bytes" if "byte" in u else "ms") + "]"] = val
            else:
                rec[k] = val
    rec["dram_bytes_per_launch"] = (rec.get("dram__bytes_read.sum [bytes]", 0) +
                                    rec.get("dram__bytes_write.sum [bytes]", 0))
    res.append(rec)
json.dump(res, open(out_json, "w"), indent=1)
for r in res:
    print(json.dumps(r, indent=1))
