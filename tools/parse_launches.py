import csv,io,sys
txt=open(sys.argv[1]).read()
rows=list(csv.DictReader(io.StringIO(txt[txt.find('"ID"'):])))
by={}
for r in rows:
    k=(int(r['ID']),r['Kernel Name'].split('(')[0][-44:])
    by.setdefault(k,{})[r['Metric Name']]=r['Metric Value']
lim=int(sys.argv[2]) if len(sys.argv)>2 else 10**9
for (i,n),m in sorted(by.items())[:lim]:
    print(i,n,m.get('gpu__time_duration.sum'),m.get('launch__grid_size'),m.get('launch__block_size'),m.get('launch__registers_per_thread'))
