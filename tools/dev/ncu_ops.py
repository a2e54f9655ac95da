"""Executed-instruction histogram by SASS opcode from an ncu source page (sass view)."""
import collections, csv, io, subprocess, sys
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
    src = d.get("Source", "")
    ex = d.get("Instructions Executed", "0").replace(",", "") or "0"
    try:
        n = float(ex)
    except ValueError:
        continue
    op = src.split()[0] if src.split() else "?"
    if op.startswith("@"):
        op = src.split()[1]
    ops[op.split(".")[0]] += n
tot = sum(ops.values())
print(f"total {tot:.4g}")
for k, v in ops.most_common(25):
    print(f"{k:12s} {v / tot * 100:5.1f}%  {v:.3g}")
