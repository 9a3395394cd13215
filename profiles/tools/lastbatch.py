import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; out=[]
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr is None or len(r)<len(hdr): continue
    d=dict(zip(hdr,r))
    name=d['Kernel Name'].split('(')[0].replace('void ','').replace('froi::','').replace('unnamed>::','')
    out.append((int(d['ID']),name,float(d['Metric Value'].replace(',',''))))
out.sort()
n=len(out)//4
tot=sum(t for _,_,t in out[-n:])
print('batch total us', round(tot/1000,1))
for i,nm,t in out[-n:]:
    print(f"{nm[:30]:30s} {t/1000:8.1f}")
