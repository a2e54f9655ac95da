"""Summarise an ncu source page by CUDA source line (stall samples, instructions executed),
attributing each SASS row to the preceding source line.
usage: python tools/ncu_lines.py report.ncu-rep [topN] [--ops]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
ops = collections.Counter()
opstall = collections.Counter()
fname = "?"
cur = None
header = None
for rec in csv.reader(io.StringIO(txt)):
    if not rec:
        continue
    if rec[0] in ("File Path", "File Name"):
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] == "Function Name":
        continue
    if rec[0] == "Line No":
        header = rec
        continue
    if header is None:
        continue
    if rec[0]:
        cur = (fname, int(rec[0]))
        agg[cur][2] = rec[1].strip()[:80]
        continue
    if len(rec) < 8 or rec[2] in ("...", ""):
        continue
    try:
        st, ins = float(rec[4]), float(rec[7])
    except ValueError:
        continue
    if cur:
        agg[cur][0] += st
        agg[cur][1] += ins
    op = rec[3].split()[0] if rec[3].split() else "?"
    if op.startswith("@"):
        op = rec[3].split()[1]
    ops[op.split(".")[0]] += ins
    opstall[op.split(".")[0]] += st
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"stall samples {ts:.0f}  instructions {ti:.4e}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]/ts*100:5.1f}% st {v[1]/ti*100:5.1f}% in  {k[0]}:{k[1]:<4} {v[2]}")
if "--ops" in sys.argv:
    print("\nopcode  %instr  %stall")
    for op, n in ops.most_common(30):
        print(f"{op:10s} {n/ti*100:6.2f} {opstall[op]/ts*100:6.2f}")
