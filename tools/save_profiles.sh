# Copy the judged evidence of the last tools/gpurun_full.sh call from gpurun_out/ into profiles/
# usage: bash tools/save_profiles.sh <tag>   (e.g. r1_v5)
set -e
tag=$1
cd "$(dirname "$0")/.."
python tools/ncu_summary.py gpurun_out/prof_lr_full.ncu-rep profiles/${tag}_lr_ncu.json > /dev/null
python tools/ncu_lines.py gpurun_out/prof_lr_full.ncu-rep 40 > profiles/${tag}_lr_source_hotspots.txt 2>&1
python tools/dev/ncu_brief.py gpurun_out/prof_lr_full.ncu-rep > profiles/${tag}_lr_brief.txt
python tools/dev/ncu_ops.py gpurun_out/prof_lr_full.ncu-rep > profiles/${tag}_lr_opcodes.txt 2>/dev/null || true
python tools/dev/ncu_stall_ops.py gpurun_out/prof_lr_full.ncu-rep > profiles/${tag}_lr_stalls.txt
TAG=$tag python - <<'PY'
import csv, collections, json
rows = list(csv.reader(open('gpurun_out/launches.csv')))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    d = dict(zip(h, r))
    if d.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    v = float(d['Metric Value'].replace(',', ''))
    u = d.get('Metric Unit', 'ns')
    ms = v / 1e6 if u == 'ns' else (v / 1e3 if u == 'us' else v)
    a = agg.setdefault(d['Kernel Name'], [0, 0.0]); a[0] += 1; a[1] += ms
tot = sum(v[1] for v in agg.values())
out = ["ncu --metrics gpu__time_duration.sum --clock-control none  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary",
       "(cold-cache, serialised per-launch times; compare shares, not absolutes)", ""]
for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"{n:3d} launches {ms:13.3f} ms total {ms / tot * 100:8.3f}%  {k[:150]}")
open('profiles/r1_launches_bench.txt', 'w').write('\n'.join(out) + '\n')
rows = list(csv.reader(open('gpurun_out/dram_bench_launch.csv')))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]; h = rows[hi]
m = {}
for r in rows[hi + 1:]:
    d = dict(zip(h, r)); m[d['Metric Name']] = float(d['Metric Value'].replace(',', ''))
rec = json.load(open('profiles/ncu_summary.json'))
import glob, os, sys
tag = os.environ.get("TAG")
v = json.load(open(f'profiles/{tag}_lr_ncu.json'))[0] if tag else {}
if v:
    rec.update({"fma_pipe_active_pct": v["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"],
                "issue_active_pct": v["smsp__issue_active.avg.pct_of_peak_sustained_active"],
                "pipe_source": f"profiles/{tag}_lr_ncu.json (ncu --set full, one 131k-pixel launch of nlem_pixels_lr)"})
rec.update({"dram_bytes_read": m['dram__bytes_read.sum'], "dram_bytes_write": m['dram__bytes_write.sum'],
            "dram_bytes_per_launch": m['dram__bytes_read.sum'] + m['dram__bytes_write.sum'],
            "gpu_time_ns_under_ncu": m['gpu__time_duration.sum']})
json.dump(rec, open('profiles/ncu_summary.json', 'w'), indent=1)
PY
tail -1 gpurun_out/bench_full.log >> profiles/r1_bench_full.jsonl
echo saved ${tag}
