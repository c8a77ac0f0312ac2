import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(list)
for r in rows[hi+1:]:
    if len(r)>vi:
        try: agg[r[ki].split('(')[0][-40:]].append(float(r[vi].replace(',','')))
        except: pass
tot=sum(sum(v) for v in agg.values())
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1]))[:12]:
    print("%-45s n=%4d  mean=%9.1f us  share=%.3f"%(k,len(v),sum(v)/len(v)/1000,sum(v)/tot))
