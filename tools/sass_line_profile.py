"""Join an ncu source-page CSV (SASS, "Instructions Executed") with nvdisasm -g line info of
the same cubin; print per-source-line instructions per unit of work.

    nvdisasm -g -c kernels.sm_100a.cubin | awk (the function) > /tmp/cub/lap12.sass
    python tools/sass_line_profile.py lap_source.csv <units> <top>
"""
import re, csv, collections, sys
cur=None; off2line={}
for ln in open('/tmp/cub/lap12.sass'):
    m=re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m: cur=(m.group(1).split('/')[-1], int(m.group(2))); continue
    m=re.search(r'/\*([0-9a-f]{4,})\*/', ln)
    if m and cur: off2line[int(m.group(1),16)]=cur
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; data=rows[2:]
ia=hdr.index("Address"); ie=hdr.index("Instructions Executed"); isamp=hdr.index("Warp Stall Sampling (All Samples)")
base=int(data[0][ia],16)
agg=collections.Counter(); samp=collections.Counter(); miss=0
for r in data:
    off=int(r[ia],16)-base
    key=off2line.get(off)
    if key is None: miss+=1; key=('?',0)
    agg[key]+=int(r[ie]); samp[key]+=int(r[isamp])
tot=sum(agg.values()); laps=float(sys.argv[2])
print("total inst/LAP", tot/laps, "missing", miss, "of", len(data))
for k,v in sorted(agg.items(), key=lambda kv:-kv[1])[:int(sys.argv[3])]:
    print(f"{k[0]}:{k[1]}  {v/laps:8.1f}/LAP  {100*v/tot:5.1f}%  stall-samples {samp[k]}")
