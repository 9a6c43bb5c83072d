import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hi]; data=[dict(zip(h,r)) for r in rows[hi+1:] if len(r)==len(h)]
per=collections.defaultdict(dict)
for d in data:
    per[(d['ID'],d['Kernel Name'].split('(')[0])][d['Metric Name']]=(d['Metric Value'],d['Metric Unit'])
scale={'ns':1e-3,'us':1,'ms':1e3,'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9,'nsecond':1e-3,'usecond':1,'msecond':1e3,'second':1e6}
agg=collections.defaultdict(lambda: collections.defaultdict(float)); cnt=collections.Counter()
for (i,name),m in per.items():
    if 'pty' not in name: continue
    cnt[name]+=1
    for k,(v,u) in m.items():
        try: x=float(v.replace(',',''))*scale.get(u,1)
        except: continue
        agg[name][k]+=x
tot=sum(a['gpu__time_duration.sum'] for a in agg.values())
print(f"{'share':>6} {'us/launch':>10} {'n':>4} {'DRAM MB':>8} {'L2 MB':>8} {'issue%':>6} {'warps%':>6} {'Minst':>7} {'bankc':>8} kernel")
for name,a in sorted(agg.items(), key=lambda x:-x[1]['gpu__time_duration.sum']):
    n=cnt[name]
    print(f"{100*a['gpu__time_duration.sum']/tot:5.1f}% {a['gpu__time_duration.sum']/n:10.1f} {n:4d} {(a['dram__bytes_read.sum']+a['dram__bytes_write.sum'])/n/1e6:8.1f} {a.get('lts__t_bytes.sum',0)/n/1e6:8.1f} {a['smsp__issue_active.avg.pct_of_peak_sustained_active']/n:6.1f} {a['sm__warps_active.avg.pct_of_peak_sustained_active']/n:6.1f} {a.get('smsp__inst_executed.sum',0)/n/1e6:7.1f} {a.get('l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',0)/n/1e6:8.2f} {name[5:70]}")
