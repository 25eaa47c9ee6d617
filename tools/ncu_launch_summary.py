import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r; continue
    if not hdr or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    key = d["ID"]
    e = data.setdefault(key, {"name": d["Kernel Name"][:60], "range": d[hdr[4]].split(":")[1] if ":" in d[hdr[4]] else "", "grid": d["Grid Size"]})
    e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
tot_t = tot_b = 0
agg = collections.defaultdict(lambda: [0, 0, 0])
for k, e in data.items():
    t = e.get("gpu__time_duration.sum", 0); b = e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)
    tot_t += t; tot_b += b
    a = agg[(e["range"], e["name"])]; a[0] += t; a[1] += b; a[2] += 1
print(f"launches {len(data)}  time {tot_t/1e3:.1f} us  dram {tot_b/1e6:.1f} MB  -> {tot_b/tot_t:.1f} GB/s")
for (rg, nm), (t, b, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{rg:8s} {nm:60s} n={c:3d} {t/1e3:9.1f} us {b/1e6:9.1f} MB {b/max(t,1):8.1f} GB/s")
