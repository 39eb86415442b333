python tools/kbench.py --graph er --n 1000000 --B 512 --T 5 --quco-only --tag c4 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^(?!.*k_stream).*' --csv --log-file gpurun_out/c4_init.csv python tools/kbench.py --graph er --n 1000000 --B 512 --T 5 --quco-only --tag c4 > /dev/null 2>&1
python3 - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c4_init.csv')))
hdr=None; agg={}
for r in rows:
    if len(r)>5 and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); t=float(d['Metric Value'].replace(',',''))
        k=d['Kernel Name'][:60]; agg.setdefault(k,[0,0]); agg[k][0]+=t; agg[k][1]+=1
for k,v in sorted(agg.items(), key=lambda kv:-kv[1][0])[:12]: print(round(v[0]/1e3/4,1),'us per solve', v[1]//4, k)
PY
