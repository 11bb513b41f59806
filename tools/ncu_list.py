"""Summarise an ncu --csv launch list (per-kernel time, DRAM bytes, bandwidth)."""
import csv
import collections
import sys

lines = open(sys.argv[1]).read().split('\n')
i = [j for j, l in enumerate(lines) if l.startswith('"ID"')][0]
d = collections.OrderedDict()
for r in csv.DictReader(lines[i:]):
    k = (int(r['ID']), r['Kernel Name'].split('(')[0].replace('void unnamed>::', '')[:48], r['Grid Size'], r['Block Size'])
    d.setdefault(k, {})[r['Metric Name']] = r['Metric Value']
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 50
for k, v in list(d.items())[:lim]:
    t = float(v.get('gpu__time_duration.sum', 'nan'))
    rb = float(v.get('dram__bytes_read.sum', 'nan'))
    wb = float(v.get('dram__bytes_write.sum', 'nan'))
    extra = ' '.join(f"{m.split('.')[0].split('__')[-1]}={val}" for m, val in v.items()
                     if not m.startswith(('gpu__time', 'dram__bytes')))
    print(f"{k[0]:3d} {k[1]:48s} {k[2]:>16s} {k[3]:>12s} {t/1e6:8.3f} ms  R {rb/1e9:6.2f} W {wb/1e9:6.2f} GB "
          f"{(rb+wb)/t:6.0f} GB/s  {extra}")
