"""Per-rank timeline of the fused multi-GPU round (libhet built with HET_TIMELINE=1)."""
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
c = het.HetCache(sum(cards), D, 0.1, 100, het.HET_LFU, rank=rank, world=world, unique_id=obj[0], max_keys_per_call=n)
lib = het.load()
lib.het_debug_timeline_p2p.argtypes = [ctypes.c_void_p]
PT = 8192
buf = np.zeros(16 * PT, np.uint64)
g = gen.grads(rank, 0, n, D, device=dev)
t = 0
while t < 6500:
    keys = gen.criteo_keys(rank, t, 500, B, cards, device=dev)
    for j in range(500):
        c.lookup(keys[j], het.HET_CLOCK_AUTO); c.update(keys[j], g, 0.01); t += 1
keys = gen.criteo_keys(rank, t, 20, B, cards, device=dev)
out = torch.empty((n, D), device=dev)
names = {0: "pb.start", 1: "pb.work", 2: "pb.pub", 3: "ln.start", 4: "ln.waited", 5: "ln.done",
         6: "pr.start", 7: "pr.work", 8: "pr.pub", 9: "ig.start", 10: "ig.waited", 11: "ig.done"}
for j in range(20):
    torch.cuda.synchronize()
    dist.barrier()
    lib.het_debug_timeline_p2p(None)
    c.lookup(keys[j], het.HET_CLOCK_AUTO, out=out)
    torch.cuda.synchronize()
    lib.het_debug_timeline_p2p(buf.ctypes.data)
    c.update(keys[j], g, 0.01)
    if j < 18:
        continue
    v = buf.reshape(16, PT).astype(np.float64)
    t0 = v[0][v[0] > 0].min()
    parts = []
    for m in sorted(names):
        x = v[m][v[m] > 0]
        if x.size:
            x = (x - t0) / 1000.0
            parts.append(f"{names[m]} {np.median(x):.1f}/{x.max():.1f}")
    print(f"rank{rank} " + " | ".join(parts), flush=True)
dist.barrier()
c.close()
