"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel count, total and mean device time, and share."""
import csv, sys, collections, re
rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith('==')]
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[1:]:
    if r[ix['Metric Name']] != 'gpu__time_duration.sum':
        continue
    name = r[ix['Kernel Name']]
    m = re.search(r'(k_[a-z0-9_]+)(<[^>]*>)?', name)
    key = (m.group(1) + (m.group(2) or '')) if m else name[:50]
    v = float(r[ix['Metric Value']].replace(',', ''))
    unit = r[ix['Metric Unit']]
    v = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}.get(unit, 1.0) * v  # -> us
    tot[key] += v; cnt[key] += 1
T = sum(tot.values())
print(f"{'kernel':48s} {'n':>4s} {'total us':>10s} {'mean us':>9s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:48]:48s} {cnt[k]:4d} {v:10.1f} {v / cnt[k]:9.1f} {100 * v / T:5.1f}%")
print(f"{'TOTAL':48s} {sum(cnt.values()):4d} {T:10.1f}")
