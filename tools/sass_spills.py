"""List local-memory spill instructions (STL/LDL) of a kernel with their source lines.

    python tools/sass_spills.py file.cubin [kernel-substring]
"""
import re
import subprocess
import sys

cubin = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
txt = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
func, line, out = None, None, []
for l in txt.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        func = m.group(1)
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
    if func and want in func and re.search(r"\b(STL|LDL)", l):
        ins = re.search(r"(STL|LDL)[^;]*", l).group(0)
        out.append(f"{line}\t{ins}")
print("\n".join(out))
print(f"{len(out)} spill instructions")
