"""Table of tools/sweep_gemm.sh output: ms per shape and plan, best starred.
    python tools/sweep_gemm.py sweep.txt"""
import collections
import re
import sys

res = collections.OrderedDict()
cur = None
for line in open(sys.argv[1]).read().splitlines():
    if line.startswith("CFG["):
        cur = line[4:-1].replace("ESGD_TC_", "") or "default"
        res[cur] = {}
        continue
    m = re.match(r"(\S+)\s.*?([\d.]+) ms", line)
    if cur and m and not line.startswith("total"):
        res[cur][m.group(1)] = float(m.group(2))
names = list(res)
print("| shape | " + " | ".join(names) + " |")
print("|---|" + "---:|" * len(names))
for sh in res.get("default", {}):
    vals = [res[c].get(sh) for c in names]
    best = min(v for v in vals if v)
    print(f"| {sh} | " + " | ".join((f"**{v:.3f}**" if v == best else f"{v:.3f}") if v else "-" for v in vals) + " |")
