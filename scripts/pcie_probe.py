"""Pinned host <-> device copy bandwidth: H2D, D2H, and both concurrently."""
import torch

n = 2 * 1024 ** 3 // 8
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d_a.copy_(h_in, non_blocking=True)
    h_out.copy_(d_b, non_blocking=True)
torch.cuda.synchronize()


def timed(fn, reps=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


gb = n * 8 / 1e9
t = timed(lambda: d_a.copy_(h_in, non_blocking=True))
print(f"H2D {gb / t * 1e3:.1f} GB/s")
t = timed(lambda: h_out.copy_(d_b, non_blocking=True))
print(f"D2H {gb / t * 1e3:.1f} GB/s")


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t = timed(both)
print(f"H2D+D2H concurrent: {2 * gb / t * 1e3:.1f} GB/s total, {t:.1f} ms for 2 x {gb:.2f} GB")
