"""Print one decode step's kernel sequence (ns) from an ncu launch list."""
import csv, re, sys
rows=list(csv.reader(open(sys.argv[1]))); which=int(sys.argv[2]) if len(sys.argv)>2 else 10
hdr=None; seq=[]
for r in rows:
    if hdr is None:
        if "Kernel Name" in r: hdr=r
        continue
    d=dict(zip(hdr,r))
    if d.get("Metric Name")!="gpu__time_duration.sum": continue
    name=re.sub(r"\(.*","",d["Kernel Name"]).replace("void ","").strip()
    v=float(d["Metric Value"].replace(",",""))*{"nsecond":1e-3,"usecond":1,"msecond":1e3}.get(d.get("Metric Unit",""),1)
    seq.append((name,v,d.get("Grid Size","")))
idx=[i for i,(n,_,_) in enumerate(seq) if n=="dm::embed_kernel"]
i0=idx[which]; i1=idx[which+1] if which+1<len(idx) else len(seq)
tot=0
for n,v,g in seq[i0:i1]:
    print(f"{n:35s} {v:9.2f} us {g}"); tot+=v
print("step total", round(tot,1), "us")
