import csv, collections, json, sys
src, out_md, out_json = sys.argv[1], sys.argv[2], sys.argv[3]
rows=list(csv.reader(open(src)))
hdr=None
per=collections.defaultdict(dict)
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr is None or len(r)<len(hdr): continue
    d=dict(zip(hdr,r))
    lid=d['ID']
    name=d['Kernel Name'].split('(')[0].replace('void ','').replace('froi::','').replace('(anonymous namespace)::','').replace('<unnamed>::','').replace('unnamed>::','')
    v=float(d['Metric Value'].replace(',',''))
    u=d['Metric Unit']
    mult={'ns':1e-9,'us':1e-6,'ms':1e-3,'nsecond':1e-9,'usecond':1e-6,'msecond':1e-3,'second':1,'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9,'KB':1e3,'MB':1e6,'GB':1e9}.get(u,1)
    per[lid]['name']=name
    per[lid][d['Metric Name']]=v*mult
agg=collections.defaultdict(lambda:{'n':0,'t':0.0,'r':0.0,'w':0.0})
for lid,d in per.items():
    a=agg[d['name']]; a['n']+=1; a['t']+=d.get('gpu__time_duration.sum',0); a['r']+=d.get('dram__bytes_read.sum',0); a['w']+=d.get('dram__bytes_write.sum',0)
tot=sum(a['t'] for a in agg.values())
lines=['| kernel | launches | total ms | share | avg us/launch | DRAM GB/s (read+write) | DRAM MB/launch |','|---|---|---|---|---|---|---|']
for k,a in sorted(agg.items(), key=lambda x:-x[1]['t']):
    lines.append(f"| `{k}` | {a['n']} | {a['t']*1e3:.2f} | {a['t']/tot:.3f} | {a['t']/a['n']*1e6:.1f} | {(a['r']+a['w'])/max(a['t'],1e-12)/1e9:.0f} | {(a['r']+a['w'])/a['n']/1e6:.1f} |")
open(out_md,'w').write('\n'.join(lines)+'\n')
fl=[k for k in agg if k.startswith('k_flow_iter')]
f=agg[fl[0]]
json.dump({'kernel': fl[0], 'launches': f['n'], 'dram_bytes_per_launch': (f['r']+f['w'])/f['n'], 'avg_duration_us_cold': f['t']/f['n']*1e6, 'source': src.split('/')[-1], 'note': 'ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none (serialised, cold cache)'}, open(out_json,'w'), indent=1)
print('\n'.join(lines[:12]))
