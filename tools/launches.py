"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
iname, ival = hdr.index('Kernel Name'), hdr.index('Metric Value')
tot, agg = 0, {}
for r in rows[1:]:
    if len(r) <= ival:
        continue
    n = r[iname][:110]
    v = float(r[ival].replace(',', ''))
    a = agg.setdefault(n, [0, 0])
    a[0] += v
    a[1] += 1
    tot += v
print(f'total {tot / 1e3:.1f} us over {len(rows) - 1} launches')
for k, (v, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f'{v / 1e3:9.1f} us {100 * v / tot:5.1f}% {c:4d}  {k}')
