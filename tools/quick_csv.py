"""Print an ncu --csv --metrics launch list as one row per kernel launch."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    data.setdefault((d['ID'], d['Kernel Name']), {})[d['Metric Name']] = d['Metric Value']
keys = None
for (i, name), v in data.items():
    if keys is None:
        keys = list(v.keys())
        print('id kernel ' + ' '.join(k.split('.')[0].replace('__', ':') for k in keys))
    short = name.split('(')[0].replace('void ', '').replace('(anonymous namespace)::', '')[-44:]
    print(i, short, ' '.join(v[k] for k in keys))
