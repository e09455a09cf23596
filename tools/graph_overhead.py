"""Event-timed replay of a graph of three near-empty kernels, with the same
L2 flush + static-input copy pattern as bench.py: the fixed cost a 3-kernel
step pays outside its kernels."""
import torch

x = torch.zeros(32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
kb = torch.zeros(3328, dtype=torch.int64, device="cuda")
src = torch.ones(3328, dtype=torch.int64, device="cuda")
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        x.add_(1.0)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    x.add_(1.0); x.mul_(1.0); x.add_(-1.0)
for _ in range(10):
    g.replay()
torch.cuda.synchronize()
ts = []
for j in range(200):
    flush.fill_(j & 0xFF)
    kb.copy_(src)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
print("3 tiny kernels, graph replay: median %.2f us, mean %.2f us" % (ts[len(ts) // 2], sum(ts) / len(ts)))
