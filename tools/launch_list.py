"""Print each launch of an `ncu --metrics gpu__time_duration.sum --csv` list in order: id, us, grid, kernel."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ii = h.index('ID')
gi = h.index('Grid Size') if 'Grid Size' in h else None
pat = sys.argv[2] if len(sys.argv) > 2 else ''
for r in rows[hi + 1:]:
    name = r[ki].replace('void ', '')
    if pat in name:
        print(f"{r[ii]:>4} {float(r[vi].replace(',', ''))/1e3:9.1f} us  {r[gi] if gi is not None else '':>16}  {name[:90]}")
