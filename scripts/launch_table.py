"""Print per-launch time / DRAM bytes from an ncu --csv launch list."""
import csv, sys
for fn in sys.argv[1:]:
    rows = list(csv.reader(open(fn)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    L = {}
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        d = L.setdefault(int(r[idi]), {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    print("==", fn)
    agg = {}
    for k in sorted(L):
        d = L[k]
        nm = d["name"].split("(")[0].replace("void ", "").replace("fasmg::", "")[:28]
        t = d.get("gpu__time_duration.sum", 0) / 1e3
        by = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e9
        if t > 50:
            print(f"  {nm:28s} {t:9.1f} us {by:7.3f} GB")
        a = agg.setdefault(nm, [0, 0.0])
        a[0] += 1; a[1] += t
    for nm, (c, t) in agg.items():
        print(f"  total {nm:28s} x{c:4d} {t/1e3:8.3f} ms")
