"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: time per kernel name."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); mi = h.index('Metric Name'); vi = h.index('Metric Value'); ii = h.index('ID')
t = defaultdict(float); c = defaultdict(set); other = defaultdict(float)
for r in rows[hi + 1:]:
    name = r[ki]
    name = name[:name.find('(')] if '(' in name else name
    name = name.replace('void ', '')[:70]
    if r[mi] == 'gpu__time_duration.sum':
        t[name] += float(r[vi].replace(',', '')); c[name].add(r[ii])
    else:
        other[(name, r[mi])] += float(r[vi].replace(',', ''))
tot = sum(t.values())
print(f"total kernel time {tot/1e3:.3f} us x1e3 over {sum(len(v) for v in c.values())} launches")
for k, v in sorted(t.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{v/1e6:9.3f} ms {100*v/tot:5.1f}% {len(c[k]):5d}x  {k}")
