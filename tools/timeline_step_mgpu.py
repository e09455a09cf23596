"""Per-rank timeline of one CUDA-graph-replayed multi-GPU step (dedup,
exchange round, update; dense all-reduce on a side stream), from the
%globaltimer marks of a HET_TIMELINE=1 build.  torchrun --nproc-per-node N."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from paper_2112_07221_b200 import het  # noqa: E402
from workload import gen  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
obj = [het.het_get_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
B, D = 128, 128
n = B * 26
cards = gen.cards_for("criteo")
if os.environ.get("TL_SCALE") == "1":   # BASELINE configs[4] per GPU: 3M rows, D = 4096
    D = 4096
    cards = gen.scaled_cards(3_000_000 * world)
c = het.HetCache(sum(cards), D, 0.1, 100, het.HET_LFU, rank=rank, world=world, unique_id=obj[0], max_keys_per_call=n)
lib = het.load()
lib.het_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
lib.het_debug_timeline_p2p.argtypes = [ctypes.c_void_p]
TLW, PTW = 8192, 8192
tl = np.zeros(32 * TLW, np.uint64)
pt = np.zeros(16 * PTW, np.uint64)
g = gen.grads(rank, 0, n, D, device=dev)
dense = gen.dense_grads(rank, 0, 1 << 20, device=dev) if world > 1 and os.environ.get("TL_DENSE", "1") == "1" else None
t = 0
while t < 6500:
    keys = gen.criteo_keys(rank, t, 500, B, cards, device=dev)
    for j in range(500):
        c.lookup(keys[j], het.HET_CLOCK_AUTO); c.update(keys[j], g, 0.01); t += 1
keys = gen.criteo_keys(rank, t, 40, B, cards, device=dev)
kbuf = keys[0].clone()
out = torch.empty((n, D), device=dev)
side = torch.cuda.Stream()
c.step(kbuf, g, out, 0.01, dense, side)
torch.cuda.synchronize()
graph = c.capture_step(kbuf, g, out, 0.01, dense)
for j in range(10):
    kbuf.copy_(keys[j]); graph.replay()
torch.cuda.synchronize()
names_tl = {0: "dd.start", 2: "dd.rank", 3: "dd.tail0", 4: "dd.end", 12: "dd.evict", 16: "up.start", 18: "up.seg",
            26: "plan.kstar", 20: "up.xdone", 19: "up.sync", 21: "up.end"}
names_pt = {0: "x.start", 1: "x.probe", 2: "x.pub", 4: "x.reqwait", 5: "x.link", 12: "p.list", 13: "p.clock",
            14: "p.rows", 7: "x.proc", 8: "x.resppub", 10: "x.respwait", 11: "x.end"}
for j in range(10, 16):
    kbuf.copy_(keys[j])
    torch.cuda.synchronize()
    dist.barrier()
    lib.het_debug_timeline(None, 32, TLW)
    lib.het_debug_timeline_p2p(None)
    torch.cuda.synchronize()
    dist.barrier()
    graph.replay()
    torch.cuda.synchronize()
    lib.het_debug_timeline(tl.ctypes.data, 32, TLW)
    lib.het_debug_timeline_p2p(pt.ctypes.data)
    if j < 13:
        continue
    a = tl.reshape(32, TLW).astype(np.float64)
    b = pt.reshape(16, PTW).astype(np.float64)
    t0 = a[0][a[0] > 0].min()
    parts = []
    for nm, arr, m in [(names_tl[k], a, k) for k in (0, 2, 3, 4, 12)] + [(names_pt[k], b, k) for k in sorted(names_pt)] + \
            [(names_tl[k], a, k) for k in (16, 18, 26, 20, 19, 21)]:
        x = arr[m][arr[m] > 0]
        if x.size:
            x = (x - t0) / 1000.0
            parts.append(f"{nm} {np.median(x):.1f}/{x.max():.1f}")
    print(f"rank{rank} " + " | ".join(parts), flush=True)
dist.barrier()
del graph
c.close()
dist.destroy_process_group()
