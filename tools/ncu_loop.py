"""Per-instruction stall listing of the hottest loop of a kernel in an ncu report (SASS source
page): instructions whose execution count is >= --frac of the maximum sweep count, in address
order, with samples and top stall reasons.  usage: python tools/ncu_loop.py rep.ncu-rep [--min=N]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ex = [int(r[ix["Instructions Executed"]]) for r in data]
# the sweep count: the most common large execution count
cnt = Counter(e for e in ex if e > 0)
big = max(cnt.items(), key=lambda kv: kv[0] * kv[1])[0]
mn = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--min=")), big // 4))
tot = 0
for k, r in enumerate(data):
    e = ex[k]
    if e >= mn:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]])
        tot += s
        top = sorted(((int(r[ix[h]]), h[6:]) for h in reasons), reverse=True)[:3]
        print(f"{k:5d} {e / big:5.2f} {s:6d} {r[ix['Source']].strip()[:70]:70s} "
              + " ".join(f"{h}:{v}" for v, h in top if v))
print("loop samples", tot, "sweep-count", big)
