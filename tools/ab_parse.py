"""Summarise an A/B log of tools/order_sweep.py / tools/sweep.py runs (max per arm)."""
import collections
import re
import sys

txt = open(sys.argv[1]).read()
arms = []
cur = None
d = collections.defaultdict(list)
for line in txt.splitlines():
    if line.startswith("== "):
        cur = line[3:]
        arm = cur.split(" N=")[0]
        if arm not in arms:
            arms.append(arm)
        continue
    m = re.match(r"N=\s*(\d+) (\S+)\s+E=.*?(\d+\.\d+) GDOF/s", line)
    if m and cur:
        d[(int(m.group(1)), "poisson c1 " + m.group(2), cur.split(" N=")[0])].append(float(m.group(3)))
        continue
    m = re.match(r"(\w+)\s+ncol=(\d) (\S+)\s+kernel.*?(\d+\.\d+) GDOF/s", line)
    if m and cur and " N=" in cur:
        arm, n = cur.split(" N=")
        d[(int(n), f"{m.group(1)} c{m.group(2)} {m.group(3)}", arm)].append(float(m.group(4)))
a, b = arms[0], arms[1]
for k in sorted(set((x, y) for x, y, _ in d)):
    va, vb = max(d[k + (a,)]), max(d[k + (b,)])
    print(f"N={k[0]:2d} {k[1]:34s} {a} {va:7.1f}  {b} {vb:7.1f}  {va / vb - 1:+.1%}")
