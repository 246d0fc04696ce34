"""Per-step (g) times / DRAM MB of the min-grid cell engine kernels from an ncu launch list."""
import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; data=rows[hi+1:]
ki=h.index('Kernel Name'); vi=h.index('Metric Value'); mi=h.index('Metric Name'); ii=h.index('ID')
per=collections.OrderedDict()
for r in data:
    per.setdefault(r[ii],[r[ki],{}])[1][r[mi]]=float(r[vi].replace(',',''))
items=list(per.values())
names=[n for n,_ in items]
starts=[i for i,n in enumerate(names) if 'k_score' in n]
s,e=(starts[-3],starts[-2])
step=-1; tab=collections.defaultdict(dict)
for n,m in items[s:e]:
    nm=n.split('(')[0].split('::')[-1]
    if 'k_mg_fill' in nm: step+=1
    if step<0 or 'k_mg' not in nm: continue
    key=nm.split('<')[0]
    tab[step][key]=tab[step].get(key,0)+m['gpu__time_duration.sum']/1e3
    tab[step][key+'_MB']=tab[step].get(key+'_MB',0)+(m.get('dram__bytes_read.sum',0)+m.get('dram__bytes_write.sum',0))/1e6
keys=['k_mg_fill','k_mg_mark','k_mg_slabcol','k_mg_slab','k_mg_pair','k_mg_dim','k_mg_query']
print('step '+' '.join(f'{k[5:]:>14}' for k in keys))
for st in sorted(tab):
    print(f'{st:4d} '+' '.join(f"{tab[st].get(k,0):7.1f}/{tab[st].get(k+'_MB',0):6.0f}" for k in keys))
