"""Fused kernels' timeline from per-warp %globaltimer marks (build with HET_TIMELINE=1).

    python tools/timeline.py [--graph]

--graph: the step (lookup + update) captured once and replayed, as bench.py
times it; otherwise eager launches.  Prints p50/max of every mark, in us from
the first dedup block's start."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2112_07221_b200 import het  # noqa: E402
from workload import gen  # noqa: E402

TLW = 8192
reddit = "--reddit" in sys.argv   # BASELINE configs[2]: 14,208 distinct node ids per step, s = 10
scale = "--scale" in sys.argv     # BASELINE configs[4] per GPU: 3M rows, D = 4096
B, D = 128, (4096 if scale else 128)
n = 14208 if reddit else B * 26
graph_mode = "--graph" in sys.argv
if scale:
    os.environ.setdefault("TL_ROWS", "3000000")
cards = gen.scaled_cards(int(os.environ["TL_ROWS"])) if os.environ.get("TL_ROWS") else gen.cards_for("criteo")
dev = torch.device("cuda", 0)
R = gen.REDDIT_ROWS if reddit else sum(cards)
c = het.HetCache(R, D, 0.1, 10 if reddit else 100, het.HET_LFU, max_keys_per_call=n)


def batch(t0, T):
    if reddit:
        return torch.stack([gen.reddit_keys(0, t0 + j, n, device=dev) for j in range(T)])
    return gen.criteo_keys(0, t0, T, B, cards, device=dev)
lib = het.load()
lib.het_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
buf = np.zeros(40 * TLW, np.uint64)
g = gen.grads(0, 0, n, D, device=dev)
t = 0
fill = 40 if reddit else 6500
while t < fill:
    keys = batch(t, 20 if reddit else 500)
    for j in range(keys.shape[0]):
        c.lookup(keys[j], het.HET_CLOCK_AUTO); c.update(keys[j], g, 0.01); t += 1
keys = batch(t, 20)
out = torch.empty((n, D), device=dev)
names = {0: "dd.start", 2: "dd.work",
         12: "dd.evict", 22: "plan.start", 7: "plan.pop", 23: "plan.end", 8: "lk.start",
         13: "lk.find", 14: "lk.install", 15: "lk.vread", 10: "lk.work", 16: "up.start", 18: "up.seg",
         11: "up.xwait", 20: "up.xdone", 19: "up.sync", 21: "up.end", 24: "plan.l2", 25: "plan.l1",
         26: "plan.kstar", 28: "lk.mpop", 29: "lk.mfstack", 30: "lk.minsert",
         37: "seg.start", 38: "seg.end", 39: "mv.end", 32: "bk.scanned", 33: "bk.scattered", 34: "bk.ranked", 35: "bk.stored", 36: "bk.keys",
         9: "x.bc", 4: "x.issued", 17: "x.words", 6: "x.written", 31: "x.atomic", 1: "dd.keys", 3: "dd.prefetch", 5: "dd.count"}
kbuf, gbuf = keys[0].clone(), g.clone()
graph = None
if graph_mode:
    c.step(kbuf, gbuf, out, 0.01)
    graph = c.capture_step(kbuf, gbuf, out, 0.01)
for j in range(20):
    torch.cuda.synchronize()
    lib.het_debug_timeline(None, 40, TLW)
    if graph is not None:
        kbuf.copy_(keys[j])
        torch.cuda.synchronize()
        lib.het_debug_timeline(None, 40, TLW)
        graph.replay()
    else:
        c.lookup(keys[j], het.HET_CLOCK_AUTO, out=out); c.update(keys[j], g, 0.01)
    torch.cuda.synchronize()
    lib.het_debug_timeline(buf.ctypes.data, 40, TLW)
    if j < 17:
        continue
    v = buf.reshape(40, TLW).astype(np.float64)
    t0 = v[0][v[0] > 0].min()
    parts = []
    for m in sorted(names, key=lambda m: np.median(v[m][v[m] > 0]) if (v[m] > 0).any() else 1e30):
        x = v[m][v[m] > 0]
        if x.size:
            x = (x - t0) / 1000.0
            if m >= 37 or m == 18:   # per-warp end times: the spread
                parts.append(f"{names[m]} p10 {np.percentile(x, 10):.1f} p50 {np.median(x):.1f} "
                             f"p90 {np.percentile(x, 90):.1f} max {x.max():.1f}")
            else:
                parts.append(f"{names[m]} p50 {np.median(x):.1f} max {x.max():.1f}")
    print(" | ".join(parts))
    print("plan", het.het_debug_eviction_plan(c.h))
