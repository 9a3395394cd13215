import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
h=rows[1]; data=rows[2:]
iE=h.index("Instructions Executed"); iS=h.index("Warp Stall Sampling (All Samples)")
c=collections.Counter(); st=collections.Counter()
for r in data:
    op=r[1].split()
    if not op: continue
    o=op[0] if not op[0].startswith('@') else op[1]
    c[o.split('.')[0]]+=int(r[iE] or 0); st[o.split('.')[0]]+=int(r[iS] or 0)
tot=sum(c.values())
print('total warp instr',tot)
for k,v in c.most_common(int(sys.argv[2]) if len(sys.argv)>2 else 25): print(k,v,round(v/tot*100,1), 'stall',st[k])
