"""Register / stack usage per kernel of the built library (cuobjdump --dump-resource-usage), filtered by a regex."""
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "--dump-resource-usage", sys.argv[1]], capture_output=True, text=True).stdout
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
name = None
rows = []
for line in out.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"REG:(\d+) STACK:(\d+)", line)
    if m and name:
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        dem = dem.split("(")[0]
        if pat is None or pat.search(dem):
            rows.append((dem, int(m.group(1)), int(m.group(2))))
        name = None
for d, r, st in sorted(rows):
    print(f"{r:4d} {st:4d} {d}")
