"""SURVEY §8(f) NEXT-2 / NEXT-3 measurements on the production kernels.

  python tools/next_sweeps.py miss            # NEXT-2, one GPU
  python tools/next_sweeps.py light           # NEXT-2 light-LFU vs LFU, one GPU
  torchrun --nproc-per-node N tools/next_sweeps.py comm   # NEXT-3, N GPUs

miss: Criteo-shaped WDL keys (BASELINE configs[1] shape), cache size 3/5/10/15 %
  of the table, LFU vs LRU (P:742-749, P:761-762 Fig. cache_miss trend, on
  synthetic Zipf instead of ogbn-mag).  Each point: WARM steps from a cold
  cache, then MEAS steps counted; miss rate = (misses + expired refetches) /
  unique keys looked up, from the library's own counters.
comm: DCN-shaped (BASELINE configs[3]) at N GPUs: staleness s in {0, 10, 100,
  inf} with a 10 % cache, and the no-cache "HET Hybrid" mode (cache_frac = 0,
  R10: every key fetched, every dirty row pushed every step).  Per
  point: embedding bytes sent per step per GPU (bytes_emb_tx + bytes_clock_tx)
  and device-timed step time (lookup + update, CUDA graph, L2 flushed between
  steps); the reduction ratio and speedup are against the no-cache row
  (the paper's 88 % / 4.36-5.14x, measured here on NVLink).
Writes one JSON object per line to stdout (rank 0).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2112_07221_b200 import het  # noqa: E402
from workload import gen  # noqa: E402

B, D, F = 128, 128, 26
N_KEYS = B * F
CARDS = gen.cards_for("criteo")
R = sum(CARDS)


def miss_sweep():
    dev = torch.device("cuda", 0)
    warm, meas = int(os.environ.get("WARM", 6000)), int(os.environ.get("MEAS", 1000))
    g = gen.grads(0, 0, N_KEYS, D, device=dev)
    for frac in (0.03, 0.05, 0.10, 0.15):
        for pol, name in ((het.HET_LFU, "LFU"), (het.HET_LRU, "LRU")):
            c = het.HetCache(R, D, frac, 100, pol, max_keys_per_call=N_KEYS)
            t = 0
            t0 = time.time()
            while t < warm + meas:
                if t == warm:
                    torch.cuda.synchronize()
                    s0 = c.stats()
                keys = gen.criteo_keys(0, t, 500, B, CARDS, 0.7, device=dev)
                for j in range(min(500, warm + meas - t)):
                    c.lookup(keys[j], het.HET_CLOCK_AUTO)
                    c.update(keys[j], g, 0.01)
                    t += 1
                    if t == warm:
                        break
            torch.cuda.synchronize()
            s1 = c.stats()
            d = {k: s1[k] - s0[k] for k in ("unique", "hits", "exp1", "exp2", "misses", "evictions")}
            print(json.dumps({"sweep": "NEXT-2 miss rate", "cache_frac": frac, "policy": name, "s": 100,
                              "warm_steps": warm, "measured_steps": meas,
                              "miss_rate": (d["misses"] + d["exp1"] + d["exp2"]) / d["unique"],
                              "cold_miss_rate": d["misses"] / d["unique"], "unique_per_step": d["unique"] / meas,
                              "evictions_per_step": d["evictions"] / meas, "wall_s": round(time.time() - t0, 1)}),
                  flush=True)
            c.close()


def light_sweep():
    """Light-LFU (R27) against exact LFU on the WDL-shaped stream:
    miss rate (the paper: "similar miss rate") and the device time of a
    lookup+update step (the paper: "significantly small run-time cost"),
    CUDA events around MEAS stream-launched steps after WARM warm-up steps."""
    dev = torch.device("cuda", 0)
    warm, meas = int(os.environ.get("WARM", 6000)), int(os.environ.get("MEAS", 1000))
    g = gen.grads(0, 0, N_KEYS, D, device=dev)
    for frac in (0.03, 0.10):
        for pol, name in ((het.HET_LFU, "LFU"), (het.HET_LIGHT_LFU, "light-LFU(64)")):
            c = het.HetCache(R, D, frac, 100, pol, max_keys_per_call=N_KEYS, pin_threshold=64)
            keys = gen.criteo_keys(0, 0, warm + meas, B, CARDS, 0.7, device=dev)
            for t in range(warm):
                c.lookup(keys[t], het.HET_CLOCK_AUTO)
                c.update(keys[t], g, 0.01)
            torch.cuda.synchronize()
            s0 = c.stats()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for t in range(warm, warm + meas):
                c.lookup(keys[t], het.HET_CLOCK_AUTO)
                c.update(keys[t], g, 0.01)
            e1.record()
            torch.cuda.synchronize()
            s1 = c.stats()
            d = {k: s1[k] - s0[k] for k in ("unique", "hits", "exp1", "exp2", "misses", "evictions")}
            print(json.dumps({"sweep": "NEXT-2 light-LFU", "cache_frac": frac, "policy": name, "s": 100,
                              "warm_steps": warm, "measured_steps": meas,
                              "miss_rate": (d["misses"] + d["exp1"] + d["exp2"]) / d["unique"],
                              "pinned": s1["pinned"], "capacity": s1["capacity"],
                              "us_per_step_stream": e0.elapsed_time(e1) / meas * 1e3}), flush=True)
            c.close()


def comm_sweep():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    torch.distributed.init_process_group("nccl", device_id=dev)
    warm, meas = int(os.environ.get("WARM", 6500)), int(os.environ.get("MEAS", 200))
    g = gen.grads(rank, 0, N_KEYS, D, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    align = torch.zeros(1, device=dev)
    rows = []
    for frac, s in ((0.0, 0), (0.1, 0), (0.1, 10), (0.1, 100), (0.1, het.HET_S_INF)):
        obj = [het.het_get_unique_id() if rank == 0 else None]   # one NCCL id per communicator
        torch.distributed.broadcast_object_list(obj, src=0)
        c = het.HetCache(R, D, frac, s, het.HET_LFU, rank=rank, world=world, unique_id=obj[0], max_keys_per_call=N_KEYS)
        t = 0
        while t < warm:
            keys = gen.criteo_keys(rank, t, 500, B, CARDS, 0.7, device=dev)
            for j in range(min(500, warm - t)):
                c.lookup(keys[j], het.HET_CLOCK_AUTO)
                c.update(keys[j], g, 0.01)
                t += 1
        keys = gen.criteo_keys(rank, t, meas + 1, B, CARDS, 0.7, device=dev)
        kbuf = keys[0].clone()
        out = torch.empty((N_KEYS, D), device=dev)
        c.step(kbuf, g, out, 0.01)
        torch.cuda.synchronize()
        graph = c.capture_step(kbuf, g, out, 0.01)
        torch.cuda.synchronize()
        torch.distributed.barrier()
        s0 = c.stats()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(meas)]
        for j in range(meas):
            kbuf.copy_(keys[1 + j])
            flush.fill_(j & 0xFF)
            torch.distributed.all_reduce(align)
            ev[j][0].record()
            graph.replay()
            ev[j][1].record()
        torch.cuda.synchronize()
        s1 = c.stats()
        ms = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / meas], device=dev)
        torch.distributed.all_reduce(ms, op=torch.distributed.ReduceOp.MAX)
        tx = (s1["bytes_emb_tx"] - s0["bytes_emb_tx"] + s1["bytes_clock_tx"] - s0["bytes_clock_tx"]) / meas
        tot = torch.tensor([tx], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tot)
        d = {k: s1[k] - s0[k] for k in ("unique", "hits", "exp1", "exp2", "misses")}
        rows.append({"cache_frac": frac, "s": "inf" if s == het.HET_S_INF else s,
                     "bytes_sent_per_step_per_gpu": tot.item() / world, "ms_per_step": ms.item(),
                     "hit_rate_rank0": d["hits"] / max(d["unique"], 1)})
        del graph
        torch.cuda.synchronize()
        c.close()
    if rank == 0:
        base = rows[0]
        for r in rows:
            r.update({"sweep": "NEXT-3 comm", "n_gpus": world, "workload": "DCN-shaped, batch 128/GPU",
                      "byte_reduction_vs_nocache": 1 - r["bytes_sent_per_step_per_gpu"] / base["bytes_sent_per_step_per_gpu"],
                      "speedup_vs_nocache": base["ms_per_step"] / r["ms_per_step"]})
            print(json.dumps(r), flush=True)
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()


if __name__ == "__main__":
    {"miss": miss_sweep, "light": light_sweep, "comm": comm_sweep}[sys.argv[1]]()
