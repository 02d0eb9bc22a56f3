import csv,sys
from collections import defaultdict
agg=defaultdict(lambda:[0,0,0,""]); cur="?"; hdr=None
def fl(x):
    try: return float(x)
    except: return 0.0
for row in csv.reader(open(sys.argv[1])):
    if not row: continue
    if row[0]=="File Path": cur=row[1].split('/')[-1]; continue
    if row[0]=="Function Name": continue
    if row[0]=="Line No": hdr=row; continue
    if hdr is None: continue
    try: line=int(row[0])
    except: continue
    g=lambda n: fl(row[hdr.index(n)])
    a=agg[(cur,line)]; a[0]+=g("Instructions Executed"); a[1]+=g("Thread Instructions Executed"); a[2]+=g("Warp Stall Sampling (All Samples)"); a[3]=row[1][:80]
ti=sum(v[0] for v in agg.values()); ts=sum(v[2] for v in agg.values())
print(ti,ts)
key = 0 if len(sys.argv)<3 else int(sys.argv[2])
for (f,l),(i,t,s,src) in sorted(agg.items(), key=lambda kv:-kv[1][key])[:50]:
    print(f"{f}:{l:<5} inst%={100*i/ti:5.2f} thr={t/max(i,1):5.1f} samp%={100*s/ts:5.2f} {src}")
