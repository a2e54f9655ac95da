"""The bench's reference arm (driver contract: `bench.py --impl reference`) times the FP64 oracle
on the host and must not load the product library (its inputs come from the oracle-side
generator); its config dict is the one the GPU arm prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import io, json, runpy, sys, contextlib
sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0']
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    runpy.run_path('bench.py', run_name='__main__')
maps = open('/proc/self/maps').read()
print(json.dumps({'line': buf.getvalue().strip().splitlines()[-1],
                  'product_loaded': 'libnlem_b200' in maps,
                  'oracle_loaded': 'libnlem_oracle' in maps}))
"""


def test_reference_arm_loads_only_the_oracle():
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, capture_output=True, text=True,
                       timeout=600, check=True)
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["oracle_loaded"] and not res["product_loaded"]
    line = json.loads(res["line"])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    sys.path.insert(0, ROOT)
    import bench

    assert line["config"] == bench.bench_config(1)
