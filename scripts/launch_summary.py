import csv, sys
from collections import defaultdict
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; data=[dict(zip(h,r)) for r in rows[1:]]
k=defaultdict(dict)
for d in data:
    k[(int(d['ID']),d['Kernel Name'][:60])][d['Metric Name']]=d['Metric Value']
items=sorted(k.items())
for (i,n),m in items[-int(sys.argv[2]) if len(sys.argv)>2 else 0:]:
    print(i, n, m.get('gpu__time_duration.sum'), m.get('smsp__inst_executed.sum'), m.get('sm__warps_active.avg.pct_of_peak_sustained_active'))
