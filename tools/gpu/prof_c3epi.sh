python tools/prof_dense.py --T 3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_epi.csv python tools/prof_dense.py --T 3 > /dev/null 2>&1
python3 - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c3_epi.csv')))
hdr=None
for r in rows:
    if len(r)>5 and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        t=float(d['Metric Value'].replace(',',''))
        if t>50000: print(d['ID'], d['Kernel Name'][:70], d['Grid Size'], d['Block Size'], round(t/1e3,1),'us')
PY
