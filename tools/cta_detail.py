import numpy as np, sys
rec = np.load(sys.argv[1]); rec = rec[rec[:,0]>0]
rec = rec[(rec[:,3]&15)!=13]; rec = rec[(rec[:,3]>>62)==0]
t0 = rec[:,0].min(); seq = rec[:,3]>>4
order = np.argsort(seq, kind='stable'); rec, seq = rec[order], seq[order]
b = np.flatnonzero(np.diff(seq))+1
L = np.split(rec, b)
# find draft head launches: gemm class with grid 393 and the following gemm grid 192
idx = [i for i,r in enumerate(L) if (r[0,3]&15)==1 and len(r)==393]
print("head-like launches", len(idx))
mid = idx[len(idx)//2]
for j in range(mid-4, mid+3):
    r = L[j]; s0 = r[:,0].min()
    st = (r[:,0]-s0)/1e3; en = (r[:,1]-s0)/1e3; dur = en-st
    cnt = np.bincount(r[:,2], minlength=148)
    print(f"launch {j-mid:+d} cls={r[0,3]&15} grid={len(r)} span={en.max():.1f} sms={np.count_nonzero(cnt)} per-SM hist={np.bincount(cnt)}")
    print("   start pct", np.percentile(st,[0,25,50,75,90,100]).round(1), " dur pct", np.percentile(dur,[0,10,50,90,100]).round(1))
    print("   end pct", np.percentile(en,[0,10,50,90,100]).round(1))
r = L[mid]; s0 = r[:,0].min()
# SM occupancy over time for head
ts = np.arange(0, (r[:,1].max()-s0)/1e3, 2.0)
act = [(((r[:,0]-s0)/1e3<=t)&((r[:,1]-s0)/1e3>t)).sum() for t in ts]
sms = [len(np.unique(r[((r[:,0]-s0)/1e3<=t)&((r[:,1]-s0)/1e3>t),2])) for t in ts]
print("head active CTAs / SMs over time (2us):", list(zip(act, sms)))

base = L[mid-9][:,0].min()
print("\nabsolute (us from base): launch, grid, sms, start[min,med,max], end[min,med,max]")
for j in range(mid-9, mid+8):
    r = L[j]; st=(r[:,0]-base)/1e3; en=(r[:,1]-base)/1e3
    print(f"{j-mid:+3d} cls={r[0,3]&15} grid={len(r):4d} sms={len(np.unique(r[:,2])):3d} start {st.min():7.1f} {np.median(st):7.1f} {st.max():7.1f}  end {en.min():7.1f} {np.median(en):7.1f} {en.max():7.1f}")

# main layer: attention launches with grid 148
am = [i for i,r in enumerate(L) if (r[0,3]&15)==2 and len(r)==148]
m0 = am[len(am)//2]
base = L[m0][:,0].min()
print("\nmain layer absolute (us): launch, grid, sms, start[min,med,max], end[min,p10,med,p90,max], per-SM hist")
for j in range(m0-1, m0+7):
    r = L[j]; st=(r[:,0]-base)/1e3; en=(r[:,1]-base)/1e3
    print(f"{j-m0:+3d} cls={r[0,3]&15} grid={len(r):4d} sms={len(np.unique(r[:,2])):3d} start {st.min():7.1f} {np.median(st):7.1f} {st.max():7.1f}  end {en.min():7.1f} {np.percentile(en,10):7.1f} {np.median(en):7.1f} {np.percentile(en,90):7.1f} {en.max():7.1f} dur med {np.median(en-st):6.1f} {np.bincount(np.bincount(r[:,2],minlength=148))}")
