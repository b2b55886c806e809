"""Read-bandwidth reference points for a C2-sized array (128 MiB int64): torch
reductions and copies, CUDA events, L2 flushed by reading 512 MB before each
call."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench

    x = bench.make_input("c2", "cuda")
    y = torch.empty_like(x)
    flush = torch.ones(64 * 2**20, dtype=torch.float64, device="cuda")
    nb = x.numel() * 8
    for name, fn, byt in (("amax (read)", lambda: x.amax(), nb), ("sum dim=-1 (read)", lambda: x.amax(dim=-1), nb),
                          ("copy (read+write)", lambda: y.copy_(x), 2 * nb), ("fill (write)", lambda: y.fill_(7), nb)):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(20):
            flush.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        print(f"{name:20s} {ms * 1e3:8.1f} us  {byt / ms / 1e6:8.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
