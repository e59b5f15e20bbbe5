#!/bin/bash
# per-kernel time totals of one bench run under ncu (cold-cache, serialised): $@ = bench args
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lt.csv python bench.py "$@" > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/lt.csv')) if len(r)>5]
hdr=rows[0]; ix={h:i for i,h in enumerate(hdr)}
tot={}; cnt={}
for r in rows[1:]:
    if r[ix['Metric Name']]!='gpu__time_duration.sum': continue
    k=r[ix['Kernel Name']][:60]; tot[k]=tot.get(k,0)+float(r[ix['Metric Value']]); cnt[k]=cnt.get(k,0)+1
T=sum(tot.values())
for k,v in sorted(tot.items(), key=lambda kv:-kv[1])[:6]: print(f"{v/T*100:5.1f}% {v/1e3:9.1f} us n={cnt[k]} mean {v/cnt[k]/1e3:8.1f} us {k}")
PY
