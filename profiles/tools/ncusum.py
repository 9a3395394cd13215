import sys,csv,subprocess
want=['Duration','DRAM Throughput','Memory Throughput','L1/TEX Cache Throughput','L2 Cache Throughput','Compute (SM) Throughput','Issue Slots Busy','Executed Ipc Active','Registers Per Thread','Achieved Occupancy','Theoretical Occupancy','Eligible Warps Per Scheduler','Warp Cycles Per Issued Instruction','L1/TEX Hit Rate','L2 Hit Rate','Grid Size','Block Size','Dynamic Shared Memory Per Block']
for f in sys.argv[1:]:
    out=subprocess.run(['ncu','-i',f,'--page','details','--csv'],capture_output=True,text=True).stdout
    r=list(csv.reader(out.splitlines()))
    h=r[0]
    vals={}
    for row in r[1:]:
        if len(row)<15: continue
        name,unit,val=row[12],row[13],row[14]
        if name in want and name not in vals: vals[name]=(val,unit)
    print(f.split('_',1)[1].replace('.ncu-rep',''), ' '.join(f"{k.split()[0]}{'_'+k.split()[1] if len(k.split())>1 else ''}={v[0]}{v[1]}" for k,v in vals.items()))
    hp=[row[17][:220] for row in r[1:] if len(row)>=18 and row[15] in('HighPipeUtilization','CPIStall') ]
    for x in hp[:2]: print('   ',x)
