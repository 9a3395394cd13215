import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None
agg=collections.defaultdict(lambda:{'n':0,'t':0.0,'b':0.0})
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr is None or len(r)<len(hdr): continue
    d=dict(zip(hdr,r))
    name=d['Kernel Name'].split('(')[0].replace('void ','').replace('froi::','').replace('<unnamed>::','')
    v=float(d['Metric Value'].replace(',',''))
    m=d['Metric Name']; u=d['Metric Unit']
    mult={'nsecond':1e-3,'usecond':1,'msecond':1e3,'second':1e6,'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}.get(u,1)
    if m=='gpu__time_duration.sum': agg[name]['t']+=v*mult; agg[name]['n']+=1
    elif m.startswith('dram__bytes'): agg[name]['b']+=v*mult
tot=sum(a['t'] for a in agg.values())
print('total kernel ms', round(tot/1e3,2))
for k,a in sorted(agg.items(), key=lambda x:-x[1]['t']):
    print(f"{k[:34]:34s} n={a['n']:4d} ms={a['t']/1e3:8.2f} share={a['t']/tot:5.3f} GB/s={a['b']/max(a['t'],1e-9)/1e3:7.0f}")
