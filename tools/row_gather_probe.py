"""Probe: does a random-row gather over a multi-GB table run slower than the
same bytes from a small table (TLB reach)?  torch.index_select, CUDA events,
L2 flushed before each launch.  Usage: python tools/row_gather_probe.py"""
import torch


def timed(fn, flush, reps=20):
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    for D in (4096, 1024, 128):
        for rows_big in (300_000, 3_000_000 if D <= 1024 else 1_200_000):
            big = torch.empty(rows_big, D, device=dev)
            small = torch.empty(4096, D, device=dev)
            n = (28 << 20) // (D * 4)
            g = torch.Generator(device="cpu").manual_seed(0)
            ib = torch.randperm(rows_big, generator=g)[:n].to(dev)
            isq = torch.randint(0, 4096, (n,), generator=g).to(dev)
            out = torch.empty(n, D, device=dev)
            tb = timed(lambda: torch.index_select(big, 0, ib, out=out), flush)
            ts = timed(lambda: torch.index_select(small, 0, isq, out=out), flush)
            by = 2 * n * D * 4
            print(f"D={D} n={n} table={rows_big * D * 4 / 1e9:.1f} GB: {tb * 1e3:.1f} us ({by / tb / 1e6:.0f} GB/s)  "
                  f"small table: {ts * 1e3:.1f} us ({by / ts / 1e6:.0f} GB/s)", flush=True)
            del big, small
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
