import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if not hdr or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    e = data.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0][-50:], "grid": d["Grid Size"]})
    try: e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    except ValueError: pass
ids = list(data.keys())
half = len(ids) // 2     # second factor = second half of the launches
sel = [data[i] for i in ids[half:]]
tot = sum(e.get("gpu__time_duration.sum", 0) for e in sel)
print(f"launches {len(sel)} (of {len(ids)})  kernel time {tot/1e6:.3f} ms")
agg = collections.defaultdict(lambda: [0.0, 0, 0.0])
for e in sel:
    t = e.get("gpu__time_duration.sum", 0)
    a = agg[e["name"]]; a[0] += t; a[1] += 1; a[2] += t * e.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", 0)
for nm, (t, c, w) in sorted(agg.items(), key=lambda x: -x[1][0])[:16]:
    print(f"{nm:52s} n={c:5d} {t/1e6:8.3f} ms")
