import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
h=rows[1]; data=rows[2:]
iE=h.index("Instructions Executed")
blocks=[]; cur=None
for i,r in enumerate(data):
    e=int(r[iE] or 0)
    if cur and cur[1]==e: cur[2]+=1
    else:
        cur=[i,e,1]; blocks.append(cur)
tot=sum(b[1]*b[2] for b in blocks)
blocks.sort(key=lambda b:-b[1]*b[2])
for b in blocks[:int(sys.argv[2]) if len(sys.argv)>2 else 12]: print('start',b[0],'exec',b[1],'len',b[2],'share',round(b[1]*b[2]/tot,3), data[b[0]][1][:60])
