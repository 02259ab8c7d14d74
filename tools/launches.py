"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
seq = []
for r in rows[hdr + 1:]:
    if len(r) <= vi: continue
    v = float(r[vi].replace(',', '')); u = r[ui]
    v = v / 1e3 if u == 'ns' else v * 1e3 if u == 'ms' else v
    seq.append((r[ki].split('(')[0].replace('void ', '')[:48], v))
agg = collections.OrderedDict()
for n, v in seq:
    a = agg.setdefault(n, [0, 0.0]); a[0] += 1; a[1] += v
tot = sum(v for _, v in seq)
print(f"{'kernel':48s} {'n':>5s} {'total_us':>10s} {'share':>6s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:48s} {n:5d} {t:10.1f} {100*t/tot:5.1f}%")
if len(sys.argv) > 2:
    marker = sys.argv[2]
    idx = [i for i, (n, _) in enumerate(seq) if marker in n]
    if idx:
        print('--- last run from', marker)
        for n, v in seq[idx[-1]:]:
            print(f"  {n:48s} {v:9.1f}")
