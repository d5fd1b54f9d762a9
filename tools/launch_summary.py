import csv, sys, collections
def load(p):
    rows=[]
    with open(p) as f:
        lines=[l for l in f if not l.startswith('==')]
    r=csv.DictReader(lines)
    for x in r:
        if x.get('Metric Name')=='gpu__time_duration.sum':
            v=float(x['Metric Value'].replace(',',''))
            unit=x['Metric Unit']
            if unit=='usecond': v*=1e3
            elif unit=='msecond': v*=1e6
            rows.append((x['Kernel Name'],v))
    return rows
for p in sys.argv[1:]:
    rows=load(p)
    agg=collections.defaultdict(lambda:[0,0.0])
    for n,v in rows:
        k=n.split('(')[0][:90]
        agg[k][0]+=1; agg[k][1]+=v
    tot=sum(v for _,v in rows)
    print(f"== {p}: {len(rows)} launches, total {tot/1e3:.1f} us")
    for k,(c,v) in sorted(agg.items(), key=lambda x:-x[1][1]):
        print(f"{v/1e3:10.1f} us {100*v/tot:5.1f}%  n={c:4d}  {k}")
