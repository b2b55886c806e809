"""Host time of one ShardedRunner step (run under torchrun, world size 1):
at 8 GPUs a C4 rank computes ~0.4 ms per step, so the runner's Python/NCCL
overhead must stay well below that."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2106_00124_b200 as ex
from paper_2106_00124_b200 import sharded

for k, v in (("RANK", "0"), ("LOCAL_RANK", "0"), ("WORLD_SIZE", "1"), ("MASTER_ADDR", "127.0.0.1"),
             ("MASTER_PORT", "29533")):
    os.environ.setdefault(k, v)
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
for route in ("box-complement", "bdbsc", "bdbs"):
    ext, box = (128, 1024, 1024), (16, 16, 16)
    x = sharded.make_local_slab(lambda p0, p1: torch.rand((p1 - p0,) + ext[1:], device=dev), ext, 0, 1, box)
    r = sharded.ShardedRunner(route, ex.Float32AddOps(), ext, box, 0, 1, dev)
    for _ in range(5):
        r(x)
    torch.cuda.synchronize()
    n = 50
    t0 = time.perf_counter()
    for _ in range(n):
        r(x)
    host = (time.perf_counter() - t0) / n
    torch.cuda.synchronize()
    tot = (time.perf_counter() - t0) / n
    print(f"{route:15s} host {host * 1e3:.3f} ms/step, wall incl. GPU {tot * 1e3:.3f} ms/step")
dist.destroy_process_group()
