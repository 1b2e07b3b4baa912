"""Per-kernel stall-reason shares, global-load tag requests by instruction and the top stalled SASS
instructions of an ncu report (source page).  usage: python tools/ncu_stalls.py REPORT.ncu-rep"""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# find last kernel section
secs=[i for i,r in enumerate(rows) if r and r[0]=="Kernel Name"]
start=secs[-1]
hdr=rows[start+1]; H={h:i for i,h in enumerate(hdr)}
data=rows[start+2:]
reasons=[h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot=sum(int(r[H["# Samples"]]) for r in data if len(r)>10)
print("total samples",tot)
agg={h:0 for h in reasons}
for r in data:
    if len(r)<10: continue
    for h in reasons: agg[h]+=int(r[H[h]])
print({k:round(100*v/tot,1) for k,v in sorted(agg.items(), key=lambda kv:-kv[1])[:8]})
# global load stats
tag=0; sect=0; ideal=0
per=[]
for idx,r in enumerate(data):
    if len(r)<10: continue
    t=int(r[H["L1 Tag Requests Global"]]); s=int(r[H["L2 Theoretical Sectors Global"]])
    if t or s: per.append((t,s,int(r[H["Instructions Executed"]]),r[H["Source"]].strip(), r[H["Access Size"]]))
    tag+=t; sect+=s
print("L1 tag requests global",tag,"theoretical sectors",sect)
for p in sorted(per,reverse=True)[:16]: print(p)
print("--- top stall instrs")
top=sorted([r for r in data if len(r)>10], key=lambda r:-int(r[H["# Samples"]]))[:25]
for r in top:
    rs=sorted(((int(r[H[h]]),h) for h in reasons),reverse=True)[:2]
    print(r[H["# Samples"]], r[H["Instructions Executed"]], r[H["Source"]].strip()[:60], rs)
print("--- tags by access kind")
from collections import defaultdict
d=defaultdict(lambda:[0,0,0])
for t,s,i,src,sz in per:
    key=src.split()[0 if not src.startswith('@') else 1]
    d[key][0]+=t; d[key][1]+=s; d[key][2]+=i
for k,v in sorted(d.items(), key=lambda kv:-kv[1][0]): print(k, v)
