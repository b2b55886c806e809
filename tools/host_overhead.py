"""Host-side cost of one small route call (C1-sized), and where it goes."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_00124_b200 as ex

x = torch.rand(1024, 1024, dtype=torch.float64, device="cuda")
t = ex.Tensor(ex.FloatAddOps(), x)
for _ in range(50):
    ex.bdbs_included(t, (32, 32))
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for _ in range(n):
    ex.bdbs_included(t, (32, 32))
host = (time.perf_counter() - t0) / n
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / n
print(f"host per call {host * 1e6:.1f} us, with sync amortised {tot * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(500):
    ex.bdbs_included(t, (32, 32))
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
