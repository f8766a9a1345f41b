import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
st = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
h = rows[st]; ki = h.index('Kernel Name'); mi = h.index('Metric Name'); vi = h.index('Metric Value')
d = collections.defaultdict(list)
for r in rows[st + 1:]:
    d[(r[ki].split('(')[0], r[mi])].append(float(r[vi].replace(',', '')))
for k, v in d.items():
    print(k, 'n', len(v), 'min', min(v), 'median', sorted(v)[len(v) // 2])
