import csv, collections, subprocess, sys
rep=sys.argv[1]
out=subprocess.run(["ncu","-i",rep,"--page","details","--csv"],capture_output=True,text=True).stdout
for line in out.splitlines():
    p=line.split('","')
    if len(p)<4: continue
    key=p[-4]+" | "+p[-3]
    if any(k in key for k in ["| Duration","DRAM Throughput","Registers Per","Achieved Occupancy","Executed Ipc Active","Issue Slots Busy","Warp Cycles Per Issued","Grid Size","L2 Hit Rate","L1/TEX Hit"]):
        print(key, p[-1][:-2] if p[-1].endswith('",') else p[-1])
    if "FP64 peak" in line or "highest-utilized" in line: print("   ", p[-4][:160])
sass=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source=sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(sass.splitlines()))
hdr=rows[1]; idx={h:i for i,h in enumerate(hdr)}
data=[]
for r in rows[2:]:
    if r and r[0]=="Kernel Name": break
    if len(r)>=len(hdr): data.append(r)
def f(r,k):
    try: return float(r[idx[k]])
    except: return 0.0
tot=sum(f(r,"Instructions Executed") for r in data); ts=sum(f(r,"Warp Stall Sampling (All Samples)") for r in data)
op=collections.Counter(); ops=collections.Counter()
for r in data:
    w=r[idx["Source"]].split()
    if not w: continue
    o=w[1] if w[0].startswith("@") else w[0]
    o=o.split('.')[0]
    op[o]+=f(r,"Instructions Executed"); ops[o]+=f(r,"Warp Stall Sampling (All Samples)")
print("total inst executed", tot)
for o,c in op.most_common(12): print("  %-8s %5.1f%% exec %5.1f%% stall-samples"%(o,100*c/tot,100*ops[o]/ts))
st=collections.Counter()
for k in hdr:
    if k.startswith("stall_") and "Not Issued" not in k: st[k]=sum(f(r,k) for r in data)
print(" ", [(k[6:],round(100*v/ts,1)) for k,v in st.most_common(8)])
