"""Top CUDA source lines by executed warp instructions from an ncu report (dev tool): python tools/ncu_inst_lines.py <rep>."""
import collections, csv, subprocess, sys
rep=sys.argv[1]
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","cuda,sass","-k",(sys.argv[2] if len(sys.argv)>2 else "k_engine")],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
hdr=None; cur=None; agg=collections.Counter(); src={}; fn=None
for r in rows:
    if not r: continue
    if r[0]=="File Path": fn=r[1].split("/")[-1]; continue
    if r[0]=="Line No": hdr=r; ii=hdr.index("Instructions Executed"); continue
    if hdr is None or len(r)<=ii: continue
    if r[0]:
        cur=(fn,r[0]); src[cur]=r[1]
        try: agg[cur]+=float(r[ii] or 0)
        except: pass
tot=sum(agg.values())
print("total warp inst", tot)
for k,v in agg.most_common(45):
    print(f"{k[0]:22s} {k[1]:>5s} {v/tot*100:5.1f}% {src[k].strip()[:110]}")
