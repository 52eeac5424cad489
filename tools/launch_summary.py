"""Summarize an ncu --csv gpu__time_duration launch list: per-kernel totals (second half of the run)."""
import csv, collections, io, sys
txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
rows = [r for r in csv.DictReader(io.StringIO(txt)) if r['Metric Name'] == 'gpu__time_duration.sum']
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
rows = rows[int(len(rows) * (1 - frac)):]
agg = collections.OrderedDict()
for r in rows:
    k = r['Kernel Name'][:48] + ' g' + r['Grid Size']
    agg.setdefault(k, [0, 0.0])
    agg[k][0] += 1
    agg[k][1] += float(r['Metric Value']) / 1e3
tot = sum(t for c, t in agg.values())
print(f'{len(rows)} launches, total {tot / 1e3:.2f} ms')
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 14]:
    print(f'{c:6d} {t / 1e3:9.2f} ms {t / c:9.1f} us/launch {100 * t / tot:5.1f}%  {k}')
