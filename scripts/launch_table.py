"""Per-kernel table of one bench step from an ncu launch list with several metrics
(gpu__time_duration + dram bytes):  python scripts/launch_table.py launches.csv
Times are printed in ns (the csv unit)."""
import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; data=rows[hi+1:]
ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit'); mi=h.index('Metric Name'); ii=h.index('ID')
per=collections.OrderedDict()
for r in data:
    per.setdefault(r[ii],[r[ki],{}])[1][r[mi]]=(float(r[vi].replace(',','')),r[ui])
names=[v[0] for v in per.values()]
starts=[i for i,n in enumerate(names) if 'k_score' in n]
s,e=(starts[-3],starts[-2]) if len(starts)>=3 else (0,len(names))
items=list(per.values())[s:e]
tot=collections.OrderedDict()
for n,m in items:
    t,u=m['gpu__time_duration.sum']; t = t/1e3 if u=='nsecond' else (t*1e3 if u=='msecond' else t)
    b=0
    for k in ('dram__bytes_read.sum','dram__bytes_write.sum'):
        if k in m:
            v,u=m[k]; b+= v*{'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}.get(u,1)
    nm=n.split('(')[0].replace('void ','')[:70]
    a=tot.setdefault(nm,[0,0,0]); a[0]+=t; a[1]+=1; a[2]+=b
T=sum(a[0] for a in tot.values())
print("| kernel | launches/step | us/step | share | DRAM MB/step |\n|---|---|---|---|---|")
for k,a in sorted(tot.items(), key=lambda x:-x[1][0]):
    print(f"| `{k}` | {a[1]} | {a[0]:.1f} | {100*a[0]/T:.1f}% | {a[2]/1e6:.0f} |")
print(f"| **total** | {sum(a[1] for a in tot.values())} | {T:.1f} | 100% | {sum(a[2] for a in tot.values())/1e6:.0f} |")
