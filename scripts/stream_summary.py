import csv, sys
from collections import OrderedDict
for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = rows[0]
    data = [dict(zip(h, r)) for r in rows[1:]]
    k = OrderedDict()
    for d in data:
        k.setdefault((int(d['ID']), d['Kernel Name'][:40]), {})[d['Metric Name']] = float(d['Metric Value'].replace(',', ''))
    items = list(k.items())
    print(f, len(items))
    for (i, n), m in items[-7:]:
        print(i, n, m.get('gpu__time_duration.sum'), round((m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)) / 1e6, 1),
              'occ', round(m.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0), 1), 'sm%',
              round(m.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0), 1))
