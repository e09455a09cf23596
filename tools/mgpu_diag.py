"""Staged multi-GPU diagnostic: which step mode works (prints after each stage)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2112_07221_b200 import het  # noqa: E402
from workload import gen  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    stages = sys.argv[1] if len(sys.argv) > 1 else "ABCD"
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    obj = [het.het_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    cards = gen.scaled_cards(2_000_000)
    R, D, B = sum(cards), 128, 128
    n = B * 26
    c = het.HetCache(R, D, 0.1, 100, het.HET_LFU, rank=rank, world=world, unique_id=obj[0], max_keys_per_call=n)
    keys = gen.criteo_keys(rank, 0, 400, B, cards, device=dev)
    g = gen.grads(rank, 0, n, D, device=dev)
    out = torch.empty((n, D), device=dev)
    dense = torch.ones(1 << 20, device=dev)
    side = torch.cuda.Stream()
    t = 0

    def say(msg):
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            print(f"[{time.strftime('%H:%M:%S')}] {msg}", flush=True)

    say("created")
    if "A" in stages:
        for j in range(50):
            c.lookup(keys[t], het.HET_CLOCK_AUTO, out=out); c.update(keys[t], g, 0.01); t += 1
            het.het_dense_allreduce(c.h, dense, dense.numel())
        say("A eager, dense serial ok")
    if "B" in stages:
        for j in range(50):
            c.step(keys[t], g, out, 0.01, dense, side); t += 1
        say("B eager, dense on side stream ok")
    kbuf = keys[0].clone()
    gr = None
    if "C" in stages:
        gr = c.capture_step(kbuf, g, out, 0.01)
        say("C captured")
        for j in range(50):
            kbuf.copy_(keys[t]); gr.replay(); t += 1
        say("C graph without dense ok")
    if "D" in stages:
        gr = c.capture_step(kbuf, g, out, 0.01, dense)
        say("D captured")
        for j in range(50):
            kbuf.copy_(keys[t]); gr.replay(); t += 1
        say("D graph with dense ok")
    st = c.stats()
    if rank == 0:
        print("stats", st, flush=True)
    del gr
    torch.cuda.synchronize()
    dist.barrier()
    c.close()
    dist.destroy_process_group()
    if rank == 0:
        print("closed", flush=True)


if __name__ == "__main__":
    main()
