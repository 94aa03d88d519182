"""Tabulate a multi-arm A/B log written by tools/ab_sweep.py runs separated by '== ARM' lines."""
import collections
import re
import sys

d = collections.defaultdict(dict)
arms = []
cur = None
for line in open(sys.argv[1]):
    if line.startswith("=="):
        cur = line.split()[1]
        arms.append(cur) if cur not in arms else None
        continue
    m = re.match(r"(\S+)\s+(\S+)\s+([\d.]+) us", line)
    if m and cur:
        d[(m[1], m[2])].setdefault(cur, []).append(float(m[3]))
print(f"{'layer':28s} {'mode':6s} " + " ".join(f"{a:>9s}" for a in arms))
for k, v in d.items():
    best = min(min(x) for x in v.values())
    print(f"{k[0]:28s} {k[1]:6s} " + " ".join(
        f"{min(v[a]):8.1f}{'*' if a in v and min(v[a]) == best else ' '}" if a in v else " " * 9 for a in arms))
