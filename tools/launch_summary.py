import csv, collections, re, sys
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv")))
hdr = None; out = []
for r in rows:
    if "Kernel Name" in r: hdr = r; continue
    if hdr and len(r) == len(hdr): out.append(r)
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
agg = collections.defaultdict(lambda: [set(), 0.0])
for r in out:
    if r[mi] != "gpu__time_duration.sum": continue
    m = re.search(r"::(\w+)(<[^(]*>)?\(", r[ki]); key = (m.group(1) + (m.group(2) or "")) if m else r[ki][:40]
    agg[key][0].add(r[ii]); agg[key][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:60]:60s} n={len(v[0]):4d} total={v[1]/1e3:9.1f}us avg={v[1]/len(v[0])/1e3:8.2f}us {v[1]/tot*100:5.1f}%")
