"""Summarise an ncu --metrics gpu__time_duration.sum launch list by kernel (dev aid).
usage: launch_summary.py launches.csv [reps]   (the last 1/reps of the launches)"""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; data = rows[1:]
ik = h.index('Kernel Name'); iv = h.index('Metric Value')
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
def name(k):
    base = k.split('(')[0].split('::')[-1].split('<')[0]
    return base + ('<true>' if '(bool)1' in k else '')
ks = [(name(r[ik]), float(r[iv].replace(',', ''))) for r in data]
per = len(ks) // reps
agg = collections.defaultdict(lambda: [0, 0.0])
for k, v in ks[-per:]:
    agg[k][0] += 1; agg[k][1] += v
tot = sum(v for _, v in agg.values())
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:20s} {c:5d} {v / 1e6:9.3f} ms  {100 * v / tot:5.1f}%")
print("total %.3f ms" % (tot / 1e6))
