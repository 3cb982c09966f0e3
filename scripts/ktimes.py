"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel name."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[start]
iK, iV, iM = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Name')
d = collections.defaultdict(list)
for r in rows[start + 1:]:
    if len(r) > iV and r[iM] == 'gpu__time_duration.sum':
        d[r[iK].split('(')[0][-44:]].append(float(r[iV].replace(',', '')))
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{k:46s} n={len(v):4d} avg_us={sum(v)/len(v)/1e3:8.2f} total_us={sum(v)/1e3:10.1f}")
