"""Stall samples by reason, attributed to SASS opcodes (and the preceding instruction's opcode)."""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = [r for r in csv.reader(io.StringIO(txt)) if r]
hdr = next(r for r in rows if r[0] == "Address")
body = rows[rows.index(hdr) + 1:]
reasons = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
agg = collections.defaultdict(collections.Counter)
tot = collections.Counter()
prev = "?"
for r in body:
    d = dict(zip(hdr, r))
    src = d.get("Source", "").split()
    op = "?" if not src else (src[1] if src[0].startswith("@") else src[0])
    for c in reasons:
        try:
            v = float(d.get(c, "0").replace(",", "") or 0)
        except ValueError:
            v = 0
        agg[c][op] += v
        tot[c] += v
    prev = op
allt = sum(tot.values())
for c, v in tot.most_common(8):
    print(f"{c:22s} {v / allt * 100:5.1f}%   top ops: " +
          ", ".join(f"{o} {n / v * 100:.0f}%" for o, n in agg[c].most_common(5)))
