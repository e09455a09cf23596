"""Host-side cost of one host-buffer step through the C-ABI (the e2e leg):
CPU time of het_lookup / het_update calls vs the device time of the step.
WDL shapes, pinned host buffers, after a short warm-up (no cache fill: the
API's host work does not depend on the cache state).  python tools/host_overhead.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2112_07221_b200 import het  # noqa: E402
from workload import gen  # noqa: E402


def main():
    B, D = 128, 128
    n = B * 26
    cards = gen.cards_for("criteo")
    c = het.HetCache(sum(cards), D, 0.1, 100, het.HET_LFU, max_keys_per_call=n)
    T = 300
    keys = gen.criteo_keys(0, 0, T, B, cards).pin_memory()
    grads = gen.grads(0, 0, n, D).pin_memory()
    out = torch.empty((n, D), dtype=torch.float32).pin_memory()
    st = torch.cuda.current_stream()
    for t in range(50):
        het.het_lookup(c.h, keys[t], n, het.HET_CLOCK_AUTO, out)
        het.het_update(c.h, keys[t], n, grads, 0.01)
    torch.cuda.synchronize()
    cl, cu, gpu = [], [], []
    for t in range(50, T):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        a = time.perf_counter()
        het.het_lookup(c.h, keys[t], n, het.HET_CLOCK_AUTO, out)
        b = time.perf_counter()
        het.het_update(c.h, keys[t], n, grads, 0.01)
        d = time.perf_counter()
        e1.record(st)
        e1.synchronize()
        cl.append((b - a) * 1e6)
        cu.append((d - b) * 1e6)
        gpu.append(e0.elapsed_time(e1) * 1e3)
    med = lambda x: sorted(x)[len(x) // 2]
    print(f"host us: lookup {med(cl):.1f} update {med(cu):.1f}; device step us {med(gpu):.1f}")
    # the same with device buffers (no staging copies, no D2H)
    kd = keys[:T].cuda()
    gd, od = grads.cuda(), out.cuda()
    cl, cu = [], []
    for t in range(50, T):
        a = time.perf_counter()
        het.het_lookup(c.h, kd[t], n, het.HET_CLOCK_AUTO, od)
        b = time.perf_counter()
        het.het_update(c.h, kd[t], n, gd, 0.01)
        d = time.perf_counter()
        torch.cuda.synchronize()
        cl.append((b - a) * 1e6)
        cu.append((d - b) * 1e6)
    print(f"host us, device buffers: lookup {med(cl):.1f} update {med(cu):.1f}")
    # raw costs of the runtime calls the binding and the library make
    import ctypes
    x = torch.empty(8, device="cuda")
    ts = []
    for _ in range(200):
        a = time.perf_counter()
        torch.cuda.current_stream().cuda_stream
        b = time.perf_counter()
        ts.append((b - a) * 1e6)
    print(f"torch current_stream: {med(ts):.2f} us")
    ts = []
    for _ in range(200):
        a = time.perf_counter()
        het._ptr(kd[5])
        b = time.perf_counter()
        ts.append((b - a) * 1e6)
    print(f"binding _ptr(tensor): {med(ts):.2f} us")


if __name__ == "__main__":
    main()
