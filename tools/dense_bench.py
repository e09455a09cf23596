"""Dense all-reduce (het_dense_allreduce, 2^20 floats) alone: device-timed,
max over ranks.  torchrun --nproc-per-node N tools/dense_bench.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
from paper_2112_07221_b200 import het  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
obj = [het.het_get_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
c = het.HetCache(1 << 20, 128, 0.01, 100, het.HET_LFU, rank=rank, world=world, unique_id=obj[0], max_keys_per_call=4096)
x = torch.randn(1 << 20, device=dev)
for _ in range(20):
    het.het_dense_allreduce(c.h, x, x.numel())
torch.cuda.synchronize()
dist.barrier()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(200):
    het.het_dense_allreduce(c.h, x, x.numel())
b.record()
torch.cuda.synchronize()
t = torch.tensor([a.elapsed_time(b) / 200 * 1e3], device=dev)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
if rank == 0:
    print(f"N={world} NCCL_CTAS={os.environ.get('HET_NCCL_CTAS', '16')} dense all-reduce 4 MB: {t.item():.1f} us", flush=True)
c.close()
dist.destroy_process_group()
