mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x --clock-control none --kernel-name-base demangled -k regex:"k_code_fused" --csv --log-file gpurun_out/fused_list.csv python scripts/prof_fused.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/fused_list.csv')) if len(r)>10]
h=rows[0]; iid=h.index('ID'); name=h.index('Kernel Name'); mn=h.index('Metric Name'); mv=h.index('Metric Value')
d={}
for r in rows[1:]:
    d.setdefault((r[iid], r[name][:60]), {})[r[mn]]=r[mv]
for (i,n),m in d.items(): print(i, n, m)
PY
