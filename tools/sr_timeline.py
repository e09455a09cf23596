"""Heavy-key segment reduce timeline (build with HET_TIMELINE=1): runs
tools/sr_probe.py's workload once and prints, for the CTA with the most stages,
the per-stage issue / data-ready times."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from workload import gen
from paper_2112_07221_b200 import het

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
D, n = 128, B * 26
dev = torch.device("cuda", 0)
c = het.HetCache(33762577, D, 0.1, 100, het.HET_LFU, max_keys_per_call=n)
keys = gen.criteo_keys(0, 0, 3, B, gen.cards_for("criteo"), 0.7, device=dev)
g = gen.grads(0, 0, n, D, device=dev)
for j in range(3):
    c.lookup(keys[j], j); c.update(keys[j], g, 0.01)
torch.cuda.synchronize()
lib = het.load()
buf = (ctypes.c_ulonglong * (148 * 256))()
lib.het_debug_timeline_sr(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(148, 256).astype(np.int64)
t0 = a[:, 0].min()
st = a[:, 3]
print("stages per CTA: max", st.max(), "median", int(np.median(st)), "sum", st.sum())
print("CTA durations us: max %.1f median %.1f" % (((a[:, 2] - a[:, 0]) / 1e3).max(), np.median((a[:, 2] - a[:, 0]) / 1e3)))
b = int(np.argmax(st))
print("CTA", b, "start %.1f prod_done %.1f cons_done %.1f us" % ((a[b, 0] - t0) / 1e3, (a[b, 1] - t0) / 1e3, (a[b, 2] - t0) / 1e3))
for i in range(min(60, st[b])):
    iss, rdy = a[b, 4 + 2 * i], a[b, 5 + 2 * i]
    print(i, "issue %.2f ready %.2f lat %.2f" % ((iss - t0) / 1e3, (rdy - t0) / 1e3, (rdy - iss) / 1e3))
print('loop cycles of the first 12 stages:', a[b, 244:256].tolist())
c.close()
