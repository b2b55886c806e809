"""Measure pinned H2D, D2H, and both at once on two streams (1 GiB each)."""
import time, torch
n = 1 << 28  # 1 GiB of float32
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True).fill_(1)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(n, device="cuda"); d_b = torch.ones(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=3):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
def h2d():
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
def both():
    h2d(); d2h()
a, b, c = t(h2d), t(d2h), t(both)
g = 4 * n / 1e9
print(f"H2D {g/a:.1f} GB/s  D2H {g/b:.1f} GB/s  both: {2*g/c:.1f} GB/s aggregate ({c*1e3:.1f} ms vs {1e3*(a+b):.1f} serial)")
