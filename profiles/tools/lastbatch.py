"""Per-kernel durations of the last batch in an ncu launch CSV (batches start at k_denoise)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
out = []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    name = d['Kernel Name'].split('(')[0].replace('void ', '').replace('froi::', '').replace('unnamed>::', '')
    out.append((int(d['ID']), name, float(d['Metric Value'].replace(',', '')) / 1000.0))
out.sort()
starts = [i for i, (_, n, _) in enumerate(out) if n.startswith('k_denoise')]
last = out[starts[-1]:]
agg = collections.defaultdict(float)
for _, n, t in last:
    agg[n] += t
tot = sum(agg.values())
print(f'last batch: {len(last)} launches, {tot:.1f} us')
for n, t in sorted(agg.items(), key=lambda x: -x[1]):
    print(f'{n[:34]:34s} {t:8.1f} {t / tot * 100:5.1f}%')
