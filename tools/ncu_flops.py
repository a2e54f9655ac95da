"""Executed FP32 work of one kernel from an ncu capture (source page, SASS view): thread-level
flops per opcode (FFMA2 4, FADD2 / FMUL2 / FFMA 2, FADD / FMUL 1 per active thread; executed
warp instructions x 32 - predicated-off lanes are not subtracted, so this is an upper bound),
next to the FMA-pipe and issue utilisation of the raw page.

    python tools/ncu_flops.py capture.ncu-rep [out.json]
"""
import collections
import csv
import io
import json
import subprocess
import sys

FLOPS = {"FFMA2": 4, "FADD2": 2, "FMUL2": 2, "FFMA": 2, "FADD": 1, "FMUL": 1}

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
ops = collections.Counter()
hdr = None
for rec in csv.reader(io.StringIO(txt)):
    if not rec:
        continue
    if rec[0] in ("Address", "#") or "Source" in rec[:3]:
        hdr = rec
        continue
    if hdr is None:
        continue
    d = dict(zip(hdr, rec))
    src = d.get("Source", "").split()
    try:
        n = float(d.get("Instructions Executed", "0").replace(",", "") or 0)
    except ValueError:
        continue
    if not src:
        continue
    op = src[1] if src[0].startswith("@") and len(src) > 1 else src[0]
    ops[op.split(".")[0]] += n
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2])) if len(rows) > 2 else {}
units = dict(zip(rows[0], rows[1])) if len(rows) > 1 else {}


def num(k):
    try:
        return float(d.get(k, "nan").replace(",", ""))
    except ValueError:
        return float("nan")


_scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9}
dur_ns = num("gpu__time_duration.sum") * _scale.get(units.get("gpu__time_duration.sum", "nsecond"), 1.0)
flops = sum(ops[k] * 32 * f for k, f in FLOPS.items())
res = {
    "kernel": d.get("Kernel Name", "")[:160],
    "duration_ns_under_ncu": dur_ns,
    "executed_fp32_flops": flops,
    "executed_fp32_tflops_under_ncu": flops / dur_ns / 1e3 if dur_ns == dur_ns else None,
    "fp32_instructions": {k: ops[k] for k in FLOPS},
    "fma_pipe_active_pct": num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "smem_wavefronts_pct": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    "smem_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    "dram_bytes": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
    "note": "flops = executed warp instructions x 32 x flops per opcode (upper bound: inactive "
            "lanes of a partially predicated instruction are counted)",
}
print(json.dumps(res, indent=1))
if len(sys.argv) > 2:
    with open(sys.argv[2], "w") as f:
        json.dump(res, f, indent=1)
