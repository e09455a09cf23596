"""Benchmark of the HET cached-embedding hot path on B200 (driver contract).

One *step* = one pass of the whole hot path over one worker-iteration of
synthetic input: het_lookup (dedup, probe, CheckValid, sync/fetch, gather)
+ het_update (segment-reduce, SGD apply + pending, overflow eviction) and,
with N > 1, the dense all-reduce of the MLP gradients.

Default workload (the driver's lines): N = 1 -> BASELINE.json configs[1]
"WDL on Criteo-shaped synthetic": 26 Zipf(0.7) fields, 33,762,577 rows,
D = 128, batch 128, cache 10 %, s = 100, LFU.  N > 1 -> configs[3] "DCN", the
same per-GPU batch with the table hash-sharded over the GPUs (weak scaling).
`--workload reddit` = configs[2] (232,965 node ids, 14,208 distinct ids per
GPU-iteration, D = 128, s = 10); `--workload scale` = configs[4] (D = 4096,
Criteo-shaped fields scaled to 3,000,000 rows per GPU, i.e. 24M rows at N = 8).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--workload auto|wdl|dcn|reddit|scale] [--no-sweep]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from workload import gen  # noqa: E402

METRIC = "embedding rows/s (lookup+update)"
UNIT = "rows/s"
R_WDL = sum(gen.CRITEO_CARDS)
SCALE_ROWS_PER_GPU = 3_000_000          # configs[4]: 24M rows over 8 GPUs


def workload_cfg(name, world):
    """BASELINE.json configs as bench workloads (SURVEY.md §8 per-config table).
    `keys` names the generator; n = batch*fields (Criteo-shaped) or K (Reddit)."""
    base = dict(D=128, batch=128, fields=26, cache_frac=0.1, policy="LFU", lr=0.01, dense_params=1 << 20)
    if name == "auto":
        name = "wdl" if world == 1 else "dcn"
    if name in ("wdl", "dcn"):
        c = dict(base, rows=R_WDL, s=100, alpha=0.7, keys="criteo", n=128 * 26)
    elif name == "reddit":
        # GraphSAGE-shaped: 128 seeds x (1 + 10 + 100) sampled ids, all distinct
        c = dict(base, rows=gen.REDDIT_ROWS, s=10, alpha=1.0, keys="reddit", n=14208, fields=None)
    elif name == "scale":
        c = dict(base, rows=SCALE_ROWS_PER_GPU * world, D=4096, s=100, alpha=0.7, keys="scale", n=128 * 26)
    else:
        raise ValueError(name)
    c["name"] = {"wdl": "WDL", "dcn": "DCN", "reddit": "Reddit-GraphSAGE", "scale": "scale-D4096"}[name]
    c["key"] = name
    return c


DATA = {"criteo": "synthetic (seeded Zipf Criteo-shaped keys, counter-hash fp32 grads)",
        "scale": "synthetic (seeded Zipf Criteo-shaped keys over fields scaled to the table, counter-hash fp32 grads)",
        "reddit": "synthetic (seeded Zipf(1.0) Reddit-shaped node ids, all distinct per step; counter-hash fp32 grads)"}


def config_dict(world, use_dense):
    """The workload of a line -- identical in both arms (the driver compares them)."""
    R = CFG["rows"]
    return {"workload": CFG["name"], "rows": R, "D": CFG["D"], "batch_per_gpu": CFG["batch"],
            "keys_per_gpu_step": CFG["n"], "fields": CFG["fields"], "cache_frac": CFG["cache_frac"],
            "cache_entries_per_gpu": int(math.floor(CFG["cache_frac"] * R)), "s": CFG["s"],
            "policy": CFG["policy"], "zipf_alpha": CFG["alpha"],
            "dense_params": CFG["dense_params"] if world > 1 else 0,
            "parallelism": f"hash-sharded table x{world}, dp{world}",
            "phase": "steady state: cache filled to C from t = 0 before timing (GPU and oracle alike)",
            "l2": "flushed between timed steps (256 MB write outside the step events)"}


CFG = workload_cfg("wdl", 1)       # mutated by main() for the selected workload


def make_keys(rank, t0, T, device):
    """[T, n] int64 keys of worker `rank`, iterations t0..t0+T-1."""
    if CFG["keys"] == "reddit":
        return torch.stack([gen.reddit_keys(rank, t0 + j, CFG["n"], CFG["rows"], CFG["alpha"], device=device)
                            for j in range(T)])
    cards = gen.cards_for("criteo") if CFG["keys"] == "criteo" else gen.scaled_cards(CFG["rows"])
    return gen.criteo_keys(rank, t0, T, CFG["batch"], cards, CFG["alpha"], device=device)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(phase, world):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
    phase's kernel from the committed `ncu --set full` capture of this workload
    (profiles/ncu_traffic.json, written by tools/ncu_traffic.py), else None.
    Cold-cache, replayed launches: compare with `achieved`'s algorithmic bytes.
    Captures: the default workload (WDL at N = 1) and the scale workload (N = 1)."""
    key = {"WDL": "n%d", "DCN": "n%d", "scale-D4096": "scale_n%d"}.get(CFG.get("name"))
    if key is None:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        ent = t[key % world][phase]
        return float(ent["dram_bytes"])
    except Exception:
        return None


# ----------------------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, gpu):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- distributed
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def max_over_ranks(x, world, device):
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def barrier(world, device):
    if world > 1:
        torch.distributed.barrier(device_ids=[device.index])
    torch.cuda.synchronize()


# ----------------------------------------------------------------------------- algorithmic bytes
def algorithmic_bytes(kernel, s, D, n_steps, resident, phases=()):
    """Algorithmic bytes per launch of one kernel:
    the bytes the method must move, from the per-step counters s (totals over
    n_steps): n occurrences, U unique, m misses, v expired, e evictions."""
    row = 4 * D
    n, U = s["keys"] / n_steps, s["unique"] / n_steps
    m, v = s["misses"] / n_steps, (s["exp1"] + s["exp2"]) / n_steps
    e, ed = s["evictions"] / n_steps, s["dirty_pushes"] / n_steps
    if kernel == "dedup":
        return 8 * n + 8 * n + 12 * U            # keys in; inverse+perm, unique+seg_off out
    if kernel == "probe":
        return U * (8 + 12 + 8 + 4 + 8 + 4 + 5)  # key, one slot, clocks, c_g, count r/w, prim, status+entry
    if kernel == "sync_fetch":
        return (m + v) * (2 * row + 8) + v * 2 * row   # W read + v write (+ p read, W write for syncs)
    if kernel == "exchange":          # N > 1 per-phase round: the local HBM side, as sync_fetch
        return algorithmic_bytes("sync_fetch", s, D, n_steps, resident)
    if kernel == "gather":
        return U * row + n * row + 4 * n + 4 * U
    if kernel == "segreduce_apply":
        return n * row + 4 * n + U * 4 * row + 8 * U
    if kernel == "evict_select":
        # LFU bitmap path: the threshold count's block counters + bitmap words, victim keys out
        return 4 * ((CFG["rows"] + 4095) // 4096) + 16 * e
    if kernel == "evict_apply":
        # per victim: key, hash slot, entry metadata; dirty: p read, W read+write, c_g
        return e * (8 + 12 + 16) + ed * (3 * row + 8)
    if kernel == "evict":
        return 4 * ((CFG["rows"] + 4095) // 4096) + 16 * e + e * (8 + 12 + 16) + ed * (3 * row + 8)
    # fused kernels = the sum of the phases they fuse
    if kernel in ("lookup_fused", "exchange_fused"):
        # exchange_fused: the local HBM side of the round (records over NVLink not counted)
        return sum(algorithmic_bytes(k, s, D, n_steps, resident) for k in ("probe", "sync_fetch", "gather"))
    if kernel == "update_fused":
        if "seg_wide" in phases:      # wide rows: k_seg_as reduced the rows; this kernel steps clocks + evicts
            return algorithmic_bytes("evict", s, D, n_steps, resident)
        return sum(algorithmic_bytes(k, s, D, n_steps, resident) for k in ("segreduce_apply", "evict"))
    # wide rows (D >= 1024): the lookup's decisions, its row moves, the ordered segment reduce
    if kernel == "lookup_dec":
        return algorithmic_bytes("probe", s, D, n_steps, resident)
    if kernel == "lookup_mv":
        return sum(algorithmic_bytes(k, s, D, n_steps, resident) for k in ("sync_fetch", "gather"))
    if kernel == "seg_wide":
        return algorithmic_bytes("segreduce_apply", s, D, n_steps, resident)
    return None


# ----------------------------------------------------------------------------- our arm
def run_gpu(args):
    from paper_2112_07221_b200 import het

    rank, world, local = dist_env()
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=device)
    B, D, F = CFG["batch"], CFG["D"], CFG["fields"]
    n = CFG["n"]
    R = CFG["rows"]
    lr = CFG["lr"]
    uid = None
    cpu_base = CpuBaseline() if (rank == 0 and world == 1 and not args.no_cpu_baseline) else None
    if world > 1:
        obj = [het.het_get_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        uid = obj[0]
    cache = het.HetCache(R, D, CFG["cache_frac"], CFG["s"], het.HET_LFU, rank=rank, world=world,
                         unique_id=uid, max_keys_per_call=n)
    C = int(math.floor(CFG["cache_frac"] * R))

    # gradient pool: distinct seeded grads per step up to ~2 GB (cache decisions
    # do not depend on gradient values, SURVEY §8(c) "value-independence")
    W, K = args.warmup, args.steps
    G = max(4, min(W + 2 * K, int(2e9 // (n * D * 4))))
    grads_all = [gen.grads(rank, j, n, D, device=device) for j in range(G)]

    # ---- fill: run the hot path until the cache holds C entries (untimed setup)
    t = 0
    chunk = 500 if CFG["keys"] != "reddit" else 4
    fill_steps = 0
    t_fill0 = time.time()
    AUTO = het.HET_CLOCK_AUTO
    while True:
        keys_blk = make_keys(rank, t, chunk, device)
        for j in range(chunk):
            k = keys_blk[j]
            cache.lookup(k, AUTO)
            cache.update(k, grads_all[t % G], lr)
            t += 1
        fill_steps += chunk
        res = cache.stats()["resident"]
        full = 1.0 if res >= C else 0.0
        if world > 1:
            full = -max_over_ranks(-full, world, device)
        if full >= 1.0 or fill_steps >= 20000:
            break
    fill_s = time.time() - t_fill0

    # ---- inputs of the measured steps, resident in HBM before timing
    keys_all = make_keys(rank, t, W + 2 * K, device)
    dense = gen.dense_grads(rank, 0, CFG["dense_params"], device=device)   # the step's dense gradients
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)   # > 126 MB L2
    align_t = torch.zeros(1, device=device)

    def between_steps(j):
        """Outside the step events: flush L2 (256 MB write); at N > 1 re-align the
        ranks with a 1-element all-reduce, so that one rank's longer flush does
        not show up as waiting inside the other rank's exchange."""
        flush.fill_(j & 0xFF)
        if world > 1:
            torch.distributed.all_reduce(align_t)
    st = torch.cuda.current_stream()

    side = torch.cuda.Stream() if world > 1 else None
    use_dense = world > 1 and not os.environ.get("HET_BENCH_NO_DENSE")   # diagnostic switch

    def step(j):
        # dense all-reduce overlapped on a side stream (N > 1)
        cache.step(keys_all[j], grads_all[j % G], out_buf, lr, dense if use_dense else None, side)

    out_buf = torch.empty((n, D), dtype=torch.float32, device=device)
    # static input buffers of the captured step (the data loader / dense
    # backward write here; filled before each timed step, outside the events)
    kbuf = torch.empty_like(keys_all[0])
    gbuf = torch.empty_like(grads_all[0])
    use_graph = world == 1 or os.environ.get("HET_P2P", "1") != "0"   # the P2P exchange has no host sync
    clk = Clocks(local)
    t_load = time.time()
    for j in range(W):
        step(j)
    while True:                             # >= 1 s of load before the timed region (clock samples)
        torch.cuda.synchronize()
        if max_over_ranks(time.time() - t_load, world, device) >= 1.0:   # same decision on every rank
            break
        for j in range(W):
            step(j)
    graph = None
    graph_launches = None
    if use_graph:
        kbuf.copy_(keys_all[0]); gbuf.copy_(grads_all[0])
        step(0)
        l0 = cache.stats()["launches"]
        graph = cache.capture_step(kbuf, gbuf, out_buf, lr, dense if use_dense else None)
        graph_launches = cache.stats()["launches"] - l0
        for j in range(3):
            kbuf.copy_(keys_all[j]); gbuf.copy_(grads_all[j % G]); graph.replay()
    barrier(world, device)
    s0 = cache.stats()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    barrier(world, device)
    torch.cuda.cudart().cudaProfilerStart()      # `ncu --profile-from-start off` sees the timed steps only
    for j in range(K):
        between_steps(j)
        if use_graph:
            kbuf.copy_(keys_all[W + j]); gbuf.copy_(grads_all[(W + j) % G])
            ev[j][0].record(st)
            graph.replay()
            ev[j][1].record(st)
        else:
            ev[j][0].record(st)
            step(W + j)
            ev[j][1].record(st)
    barrier(world, device)
    torch.cuda.cudart().cudaProfilerStop()
    clocks = clk.stop()
    s1 = cache.stats()
    ms = sum(a.elapsed_time(b) for a, b in ev) / K
    ms = max_over_ranks(ms, world, device)
    launches = graph_launches * K if use_graph else s1["launches"] - s0["launches"]
    # the same steps launched kernel by kernel on the stream (no graph), for reference
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for j in range(K):
        between_steps(j)
        ev2[j][0].record(st)
        step(W + j)
        ev2[j][1].record(st)
    torch.cuda.synchronize()
    ms_stream = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev2) / K, world, device)
    sd = {k: s1[k] - s0[k] for k in ["keys", "unique", "hits", "exp1", "exp2", "misses", "evictions",
                                     "dirty_pushes", "lookups"]}

    # ---- per-kernel timing pass (events on the launching stream) for the roofline
    het.het_profile_enable(cache.h, True)
    het.het_profile_read(cache.h)
    p0 = cache.stats()
    for j in range(K):
        between_steps(j)
        step(W + K + j)
    torch.cuda.synchronize()
    prof = het.het_profile_read(cache.h)
    het.het_profile_enable(cache.h, False)
    p1 = cache.stats()
    pd = {k: p1[k] - p0[k] for k in sd}
    wire = {k: (p1[k] - p0[k]) / K for k in ("bytes_clock_tx", "bytes_emb_tx", "bytes_clock_rx", "bytes_emb_rx")}
    resident = p1["resident"]
    hbm, peak_kind = peaks()
    kern = {}
    for name, (tot_ms, cnt) in prof.items():
        ab = algorithmic_bytes(name, pd, D, K, resident, phases=set(prof))
        avg = tot_ms / max(cnt, 1)
        kern[name] = dict(ms_per_launch=avg, launches=cnt, share=None,
                          achieved_gbs=(ab / (avg * 1e-3) / 1e9) if ab else None)
    tot = sum(v["ms_per_launch"] * v["launches"] for v in kern.values()) or 1.0
    for v in kern.values():
        v["share"] = v["ms_per_launch"] * v["launches"] / tot
    # dominant kernel of the sparse path (the dense all-reduce runs overlapped on a side stream)
    cand = [k for k in kern if k != "dense_allreduce"]
    dom = max(cand, key=lambda k: kern[k]["share"]) if cand else None
    roof = None
    if dom:
        a = kern[dom]["achieved_gbs"]
        roof = {"bound": "hbm", "kernel": dom, "achieved": a, "peak": hbm, "unit": "GB/s",
                "frac": (a / hbm) if a else None, "traffic": ncu_traffic(dom, world), "peak_source": peak_kind}

    # ---- e2e: same steps through the C-ABI with host (pinned) buffers
    keys_h = keys_all[:W + K].cpu().pin_memory()
    grads_h = [grads_all[j % G].cpu().pin_memory() for j in range(min(W + K, G))]
    GH = len(grads_h)
    out_h = torch.empty((n, D), dtype=torch.float32).pin_memory()
    te0, te1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for j in range(max(W, 50)):                   # >= 50 warm host-buffer steps (staging buffers, page-in)
        het.het_lookup(cache.h, keys_h[j % (W + K)], n, AUTO, out_h)
        het.het_update(cache.h, keys_h[j % (W + K)], n, grads_h[j % GH], lr)
    barrier(world, device)
    e2e_ms = 0.0
    e2e_all = []
    for j in range(K):
        between_steps(j)
        te0.record(st)
        het.het_lookup(cache.h, keys_h[W + j], n, AUTO, out_h)
        het.het_update(cache.h, keys_h[W + j], n, grads_h[(W + j) % GH], lr)
        if use_dense:
            side.wait_stream(st)
            with torch.cuda.stream(side):
                het.het_dense_allreduce(cache.h, dense, dense.numel(), stream=side)
            st.wait_stream(side)
        te1.record(st)
        te1.synchronize()
        e2e_all.append(te0.elapsed_time(te1))
        e2e_ms += e2e_all[-1]
    e2e_ms = max_over_ranks(e2e_ms / K, world, device)
    e2e_med = max_over_ranks(statistics.median(e2e_all), world, device)

    value = n * world / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": DATA[CFG["keys"]],
        "config": config_dict(world, use_dense),
        "setup": {"fill_steps": fill_steps, "fill_s": round(fill_s, 1), "grad_pool": G,
                  "rank_alignment": "ranks re-aligned after the L2 flush by a 1-element all-reduce, outside the events"
                  if world > 1 else None},
        "samples_per_s": B * world / (ms * 1e-3),
        "unique_rows_per_s": sd["unique"] / K * world / (ms * 1e-3),
        "step_counters": {k: v / K for k, v in sd.items()},
        "gpu_launches": int(launches),
        "launches_per_step": launches / K,
        "cuda_graph": use_graph,
        "ms_per_step_stream_launch": ms_stream,
        "roofline": roof,
        "kernels": kern,
        "nvlink": nvlink_fraction(kern, wire, world, device) if world > 1 else None,
        "clocks": clocks,
        "e2e": {"value": n * world / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
                "ms_per_step_median": e2e_med, "value_median": n * world / (e2e_med * 1e-3),
                "warm_steps": max(W, 50),
                "h2d_bytes_per_step": n * 8 + n * D * 4, "d2h_bytes_per_step": n * D * 4},
    }
    del graph
    torch.cuda.synchronize()
    if not args.no_sweep and world == 1 and CFG["name"] == "WDL":
        line["hbm_sweep"] = run_sweep(het, device)
    barrier(world, device)
    cache.close()
    if cpu_base is not None:
        line["cpu_baseline"] = cpu_base.result()
    return line, rank, world


def nvlink_fraction(kern, wire, world, device):
    """SURVEY §8(d) %NVLink: exchange payload bytes each GPU sends per step
    (records + rows, device-counted) / the exchange kernel's mean time, against
    an NCCL all-to-all of 64 MB per GPU timed here (per-direction bytes to
    peers / time) and against 900 GB/s nominal."""
    ex = kern.get("exchange_fused") or kern.get("exchange")
    if not ex:
        return None
    n = 64 << 20
    a = torch.empty(n // 4, dtype=torch.float32, device=device)
    b = torch.empty_like(a)
    for _ in range(3):
        torch.distributed.all_to_all_single(b, a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = float("inf")
    for _ in range(3):                                 # best of 3 trials of 10 (max over ranks)
        torch.distributed.barrier()
        e0.record()
        for _ in range(10):
            torch.distributed.all_to_all_single(b, a)
        e1.record()
        torch.cuda.synchronize()
        t = min(t, max_over_ranks(e0.elapsed_time(e1) / 10 * 1e-3, world, device))
    peak = n * (world - 1) / world / t / 1e9
    sent = wire["bytes_clock_tx"] + wire["bytes_emb_tx"]
    ach = sent / (ex["ms_per_launch"] * 1e-3) / 1e9
    return {"bytes_sent_per_gpu_step": sent, "exchange_ms": ex["ms_per_launch"], "achieved_GBs": ach,
            "nccl_alltoall_64MB_GBs": peak, "frac": ach / peak, "frac_of_900_nominal": ach / 900.0}


def run_sweep(het, device):
    """n-sweep at D = 128 to the bandwidth-bound regime:
    gather and segreduce_apply %HBM at B in {1024, 8192, 32768}."""
    res = []
    hbm, _ = peaks()
    cards = gen.cards_for("criteo")
    D = CFG["D"]
    for B in [1024, 8192, 32768]:
        n = B * 26
        c = het.HetCache(CFG["rows"], D, CFG["cache_frac"], CFG["s"], het.HET_LFU, max_keys_per_call=n)
        t = 0
        steps = max(8, 40 * 128 // B)
        keys = gen.criteo_keys(0, 0, steps + 6, B, cards, CFG["alpha"], device=device)
        g = gen.grads(0, 0, n, D, device=device)
        for j in range(steps):
            c.lookup(keys[j], t); c.update(keys[j], g, CFG["lr"]); t += 1
        het.het_profile_enable(c.h, True)
        het.het_profile_read(c.h)
        s0 = c.stats()
        for j in range(5):
            c.lookup(keys[steps + j], t); c.update(keys[steps + j], g, CFG["lr"]); t += 1
        torch.cuda.synchronize()
        prof = het.het_profile_read(c.h)
        s1 = c.stats()
        sd = {k: s1[k] - s0[k] for k in ["keys", "unique", "misses", "exp1", "exp2", "evictions", "dirty_pushes"]}
        ent = {"batch": B, "n": n}
        for kname in ["gather", "segreduce_apply", "dedup", "probe", "sync_fetch", "evict_apply"]:
            if kname in prof:
                tot, cnt = prof[kname]
                ab = algorithmic_bytes(kname, sd, D, 5, s1["resident"])
                avg = tot / cnt
                ent[kname] = {"ms": avg, "GBs": ab / (avg * 1e-3) / 1e9, "frac": ab / (avg * 1e-3) / 1e9 / hbm}
        res.append(ent)
        c.close()
    return res


# ----------------------------------------------------------------------------- oracle legs
ORACLE_CORE = 0          # the oracle runs pinned to one host core (taskset -c 0)


def _pin(core):
    """Pin this process to one core; torch's CPU ops (the input generator)
    then use one thread too, instead of a pool oversubscribing that core."""
    torch.set_num_threads(1)
    try:
        os.sched_setaffinity(0, {core})
        return True
    except (AttributeError, OSError):
        return False


def oracle_steady(world, warmup, steps, budget_s, fill_budget_s=240.0, mem_budget=16e9, go=None):
    """The CPU oracle (as it stands) on the selected workload at the SAME
    protocol phase as the GPU arm: a clocks-only fill (rows not tracked) runs
    the workload's iterations from t = 0 until every worker's cache holds C
    entries -- the GPU arm's fill criterion -- then every resident entry gets
    its row (as at a Fetch) and full-D iterations follow: `warmup` untimed,
    then up to `steps` timed ones, stopping once `budget_s` is spent.  The
    N-worker simulation runs all workers in lock step on this one core.
    `go`: called between the untimed and the timed part (the bench's
    cpu_baseline waits there until the GPU timing is over).  Returns a dict."""
    from oracle.oracle import Oracle, capacity
    n, D, R = CFG["n"], CFG["D"], CFG["rows"]
    C = capacity(CFG["cache_frac"], R)
    o = Oracle(R=R, D=D, C=C, s=CFG["s"], N=world, track_div=1 << 62)
    chunk = 500 if CFG["keys"] != "reddit" else 20
    t, t0 = 0, time.perf_counter()
    full = False
    while time.perf_counter() - t0 < fill_budget_s:
        keys = [make_keys(i, t, chunk, "cpu").numpy() for i in range(world)]
        for j in range(chunk):
            o.lookup(t + j, [keys[i][j] for i in range(world)], want_out=False)
            o.update(None, CFG["lr"])
        t += chunk
        if min(o.cache_size(i) for i in range(world)) >= C:
            full = True
            break
    fill_s = time.perf_counter() - t0
    resident = sum(o.cache_size(i) for i in range(world))
    track_div = max(1, math.ceil(resident * 2 * D * 4 / mem_budget))   # rows of v and p in host memory
    o.set_track_div(track_div)
    T = warmup + steps
    keys = [make_keys(i, t, T, "cpu").numpy() for i in range(world)]
    G = max(2, min(T, int(1e9 // (n * D * 4 * world))))
    grads = [[gen.grads(i, t + j, n, D).numpy() for i in range(world)] for j in range(G)]
    for j in range(warmup):
        o.lookup(t + j, [keys[i][j] for i in range(world)])
        o.update(grads[j % G], CFG["lr"])
    if go is not None:
        go()
    s0 = o.stats(0)
    done = 0
    t1 = time.perf_counter()
    for j in range(warmup, T):
        o.lookup(t + j, [keys[i][j] for i in range(world)])
        o.update(grads[j % G], CFG["lr"])
        done += 1
        if time.perf_counter() - t1 > budget_s:
            break
    dt = time.perf_counter() - t1
    s1 = o.stats(0)
    ev = (s1["evictions"] - s0["evictions"]) / max(done, 1)
    return {"value": n * world * done / dt, "dt": dt, "done": done, "fill_steps": t, "fill_s": fill_s,
            "full": full, "resident": resident, "capacity": C * world, "track_div": track_div,
            "evictions_per_step": ev, "t0": t + warmup}


def _sample_text(r, world, warmup):
    state = ("cache full" if r["full"] else
             f"cache at {r['resident'] / r['capacity']:.0%} of C after the {r['fill_s']:.0f} s fill budget")
    rows = "full D=%d rows" % CFG["D"] if r["track_div"] == 1 else \
        f"D={CFG['D']} rows for 1/{r['track_div']} of the keys (host-memory bound)"
    return (f"{CFG['name']} iterations {r['t0']}..{r['t0'] + r['done']} after a clocks-only fill of "
            f"{r['fill_steps']} iterations ({state}, {r['evictions_per_step']:.0f} evictions/step of worker 0) "
            f"and {warmup} untimed full-row iterations; {rows}; {world} worker(s) simulated in lock step; "
            f"single-threaded C++ oracle pinned to core {ORACLE_CORE} (taskset); {r['dt']:.1f} s timed; "
            f"host: {os.cpu_count()} cores, {_cpu_model()}")


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_child_main(args):
    """`--impl oracle-child`: the cpu_baseline leg as a separate process pinned
    to ORACLE_CORE, started at the beginning of the GPU bench.  It fills, then
    prints READY and waits for GO on stdin (sent after the GPU timing), then
    times its sample and prints one JSON line."""
    pinned = _pin(ORACLE_CORE)

    def go():
        print("READY", flush=True)
        sys.stdin.readline()
    r = oracle_steady(1, 5, 2000, budget_s=15.0, go=go)
    r["pinned"] = pinned
    r["sample"] = _sample_text(r, 1, 5)
    print(json.dumps(r), flush=True)


class CpuBaseline:
    """cpu_baseline of the N = 1 GPU bench: the oracle child process fills
    while the GPU arm runs (on other cores), and times its sample after."""

    def __init__(self):
        self.p = subprocess.Popen([sys.executable, os.path.abspath(__file__), "--impl", "oracle-child",
                                   "--workload", CFG["key"]], stdin=subprocess.PIPE, stdout=subprocess.PIPE,
                                  text=True, cwd=ROOT)
        try:   # the GPU arm stays off the oracle's core
            os.sched_setaffinity(0, set(os.sched_getaffinity(0)) - {ORACLE_CORE} or {ORACLE_CORE})
        except (AttributeError, OSError):
            pass

    def _line(self, timeout):
        import select
        r, _, _ = select.select([self.p.stdout], [], [], timeout)
        return self.p.stdout.readline() if r else None

    def result(self, timeout=400.0):
        line = self._line(timeout)               # READY (the fill is over)
        if line is None or line.strip() != "READY":
            self.p.kill()
            return {"error": "oracle child failed or timed out: " + str(line).strip()}
        self.p.stdin.write("GO\n")
        self.p.stdin.flush()
        out = self._line(timeout)
        self.p.wait()
        if not out:
            return {"error": "oracle child timed out"}
        r = json.loads(out)
        return {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "oracle", "sample": r["sample"],
                "steady_state": r["full"], "evictions_per_step": r["evictions_per_step"]}


def run_reference(args):
    """The reference arm: the CPU oracle of the paper's protocol (there is no
    reference code to install), on this arm's workload and
    config at the GPU arm's protocol phase (steady state), `world` simulated
    workers, rank 0 only, pinned to one core."""
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    _pin(ORACLE_CORE)
    r = oracle_steady(world, args.warmup, args.steps, budget_s=120.0)
    ms = r["dt"] / max(r["done"], 1) * 1e3
    sample = _sample_text(r, world, args.warmup) + (
        f" (stopped after {r['done']} of {args.steps} steps: 120 s budget)" if r["done"] < args.steps else "")
    return {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": DATA[CFG["keys"]],
            "config": config_dict(world, use_dense=False),
            "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference", "oracle-child"])
    ap.add_argument("--no-cpu-baseline", action="store_true", help="skip the oracle's cpu_baseline leg")
    ap.add_argument("--no-sweep", action="store_true", help="skip the D=128 n-sweep (HBM regime)")
    ap.add_argument("--workload", default="auto", choices=["auto", "wdl", "dcn", "reddit", "scale"])
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    CFG.clear()
    CFG.update(workload_cfg(args.workload, dist_env()[1]))
    if args.impl == "oracle-child":
        oracle_child_main(args)
        return
    if args.impl == "reference":
        line = run_reference(args)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    line, rank, world = run_gpu(args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
