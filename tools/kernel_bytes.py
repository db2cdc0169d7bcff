"""Per-kernel time / DRAM bytes of one training step from an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum (steady-state step)."""
import csv,re,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=[r for r in rows if "Kernel Name" in r][0]
ii,k,mi,v,gi=(hdr.index(x) for x in ("ID","Kernel Name","Metric Name","Metric Value","Grid Size"))
per={};order=[]
for r in rows:
    if len(r)!=len(hdr) or r is hdr: continue
    if r[ii] not in per: per[r[ii]]={'name':r[k],'grid':r[gi]}; order.append(r[ii])
    per[r[ii]][r[mi]]=float(r[v].replace(',',''))
seq=[per[i] for i in order]
xs=[j for j,p in enumerate(seq) if 'head_fwd' in p['name'] or 'xent' in p['name']]
a,b=xs[-3],xs[-2]
tot=0
for p in seq[a+1:b+1]:
    n=p['name']; m=re.search(r"tc_gemm_kernel<(\d+), (?:ce::)?(\w+)", n)
    nm=f"{m.group(2)}_{m.group(1)}" if m else re.sub(r"^void |\(.*|<.*", "", n)[:60]
    t=p['gpu__time_duration.sum']/1e3; by=(p.get('dram__bytes_read.sum',0)+p.get('dram__bytes_write.sum',0))
    tot+=t
    print(f"{t:9.1f} us {by/1e6:9.1f} MB {by/t/1e6 if t else 0:6.2f} TB/s {p['grid']:14s} {nm}")
print(f"step {tot:.1f} us")
