"""Large-batch update probe: Criteo-shaped batches at B (default 32768) on the
per-phase path; prints event-timed segreduce_apply and the stats.  Run under
`ncu --metrics gpu__time_duration.sum -k regex:k_sr|k_heavy` for per-kernel
durations (serialised)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from workload import gen
from paper_2112_07221_b200 import het

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
D = 128
n = B * 26
cards = gen.cards_for("criteo")
dev = torch.device("cuda", 0)
c = het.HetCache(33762577, D, 0.1, 100, het.HET_LFU, max_keys_per_call=n)
keys = gen.criteo_keys(0, 0, steps, B, cards, 0.7, device=dev)
g = gen.grads(0, 0, n, D, device=dev)
het.het_profile_enable(c.h, True)
for j in range(steps):
    c.lookup(keys[j], j)
    c.update(keys[j], g, 0.01)
torch.cuda.synchronize()
prof = het.het_profile_read(c.h)
for k, (tot, cnt) in sorted(prof.items()):
    print(f"{k:20s} {tot / cnt * 1000:9.1f} us x{cnt}")
c.close()
