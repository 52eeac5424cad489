"""Summarize an ncu --csv capture of (gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum) per launch: per kernel+grid totals, average duration and
achieved DRAM GB/s, largest first. usage: hbm_summary.py file.csv [top]"""
import collections, csv, io, sys

txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
per = collections.OrderedDict()
for r in csv.DictReader(io.StringIO(txt)):
    v = float(r["Metric Value"].replace(",", ""))
    u = r["Metric Unit"]
    if r["Metric Name"] == "gpu__time_duration.sum":
        v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(u, 1e-3)  # -> us
    else:
        v *= {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
    per.setdefault(r["ID"], {"k": r["Kernel Name"][:44] + " g" + r["Grid Size"]})[r["Metric Name"]] = v
agg = collections.OrderedDict()
for e in per.values():
    a = agg.setdefault(e["k"], [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += e.get("gpu__time_duration.sum", 0.0)
    a[2] += e.get("dram__bytes_read.sum", 0.0)
    a[3] += e.get("dram__bytes_write.sum", 0.0)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 16
print(f"{'launches':>8} {'total ms':>9} {'us/launch':>10} {'rd MB/l':>9} {'wr MB/l':>9} {'GB/s':>8}  kernel grid")
for k, (c, t, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{c:8d} {t / 1e3:9.2f} {t / c:10.1f} {rd / c / 1e6:9.2f} {wr / c / 1e6:9.2f} {(rd + wr) / (t * 1e-6) / 1e9:8.0f}  {k}")
