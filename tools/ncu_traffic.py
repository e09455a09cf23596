"""Per-launch DRAM traffic of the hot-path kernels from an `ncu --set full`
report -> profiles/ncu_traffic.json (read by bench.py for roofline.traffic).

  python tools/ncu_traffic.py <report.ncu-rep> <n_gpus> [source-note] [workload]

workload: omitted for the default (WDL / DCN) capture, else e.g. "scale"
(stored under "<workload>_n<N>").
"""
import csv
import io
import json
import os
import subprocess
import sys

PHASE = {"k_dd_fused": "dedup", "k_lookup_fused": "lookup_fused", "k_update_fused": "update_fused",
         "k_probe_build": "exchange_fused", "k_sr_light": "segreduce_apply",
         "k_lookup_wide": "lookup_dec", "k_mv_as": "lookup_mv", "k_seg_as": "seg_wide"}

rep, world = sys.argv[1], int(sys.argv[2])
note = sys.argv[3] if len(sys.argv) > 3 else os.path.basename(rep)
workload = sys.argv[4] if len(sys.argv) > 4 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]
ik = hdr.index("Kernel Name")
acc = {}
for r in data:
    name = r[ik].split("(")[0].split("<")[0].split("::")[-1].split()[-1]
    if name not in PHASE:
        continue
    vals = {}
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        i = hdr.index(m)
        v = float(r[i].replace(",", ""))
        u = units[i]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "usecond": 1e3, "us": 1e3,
                 "msecond": 1e6}.get(u, 1)
        vals[m] = v * scale
    a = acc.setdefault(name, [0.0, 0.0, 0])
    a[0] += vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    a[1] += vals["gpu__time_duration.sum"]
    a[2] += 1
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
try:
    t = json.load(open(path))
except Exception:
    t = {}
key = ("%s_n%d" % (workload, world)) if workload else ("n%d" % world)
if workload:
    t["source_" + key] = note
else:
    t["source"] = note
ent = t.setdefault(key, {})
for name, (b, ns, cnt) in acc.items():
    ent[PHASE[name]] = {"kernel": name, "dram_bytes": b / cnt, "ncu_ns": ns / cnt, "launches": cnt}
json.dump(t, open(path, "w"), indent=1, sort_keys=True)
print(json.dumps(t, indent=1, sort_keys=True))
