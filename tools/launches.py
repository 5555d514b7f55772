import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]
ki, vi, mi = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Name')
agg = collections.defaultdict(list)
for r in rows[hdr_i+1:]:
    if len(r) > vi and r[mi] == 'gpu__time_duration.sum':
        agg[r[ki][:100]].append(float(r[vi].replace(',', '')))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):4d} {sum(v)/len(v)/1e3:10.2f} us avg  min {min(v)/1e3:8.2f} max {max(v)/1e3:8.2f}  {k}")
