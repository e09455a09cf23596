"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rows = list(csv.reader(open(path)))
hdr = None
agg = collections.OrderedDict()
dram = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    k = d["Kernel Name"].split("(")[0][:48]
    if d.get("Metric Name") in ("dram__bytes_read.sum", "dram__bytes_write.sum"):   # optional: DRAM bytes
        v = float(d["Metric Value"].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(
            d.get("Metric Unit", "byte"), 1)
        dram[k] = dram.get(k, 0.0) + v
        continue
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values())
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    extra = f"  dram {dram[k] / c / 1e6:8.2f} MB/launch {dram[k] / v:7.1f} GB/s" if k in dram else ""
    print(f"{k:48s} {c:5d} launches {v / c / 1000:9.2f} us/launch {100 * v / tot:5.1f}%{extra}")
print(f"total {tot / 1000 / steps:.2f} us per step over {steps} steps")
