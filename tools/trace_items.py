"""Summarise a trace_step.py timeline: per work item of CTA 0 (MMA issuer A): sub-tiles, the gap
from the previous item's last P to this item's Q-ready, Q-ready -> first P, mean period."""
import sys

import numpy as np

lines = open(sys.argv[1]).read().splitlines()
ev = [(int(l.split()[0]), l.split()[1], ' '.join(l.split()[2:])) for l in lines if l.strip() and not l.startswith('#')]
mma = [(c, n) for c, r, n in ev if r == 'mma']
items, cur = [], None
for c, n in mma:
    if n == 'Q rdy':
        if cur:
            items.append(cur)
        cur = {'q': c, 'p': []}
    elif cur is not None and n == 'P_A rdy':
        cur['p'].append(c)
if cur:
    items.append(cur)
prev = None
tot_sub = tot_gap = tot_first = tot_body = 0
for it in items:
    n = len(it['p'])
    if not n:
        continue
    gap = it['q'] - prev if prev else 0
    first = it['p'][0] - it['q']
    body = it['p'][-1] - it['p'][0]
    print(f"subtiles {n:3d} gap {gap:6d} Q->P0 {first:6d} period {body / max(n - 1, 1):7.0f}")
    tot_sub += n; tot_gap += gap; tot_first += first; tot_body += body
    prev = it['p'][-1]
end = max(c for c, r, n in ev)
print(f"total cycles {end}: gaps {tot_gap} ({tot_gap / end:.0%}), Q->P0 {tot_first} ({tot_first / end:.0%}),"
      f" steady {tot_body} ({tot_body / end:.0%}); sub-tiles {tot_sub}, cycles/sub-tile overall {end / tot_sub:.0f}")
