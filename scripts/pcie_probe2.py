"""Pinned host <-> device copies: one stream per direction vs each copy split
over k streams per direction (more copy engines), H2D and D2H concurrent."""
import torch

n = 2 * 1024 ** 3 // 8
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]


def run(k):
    cur = torch.cuda.current_stream()
    for s in streams[:2 * k]:
        s.wait_stream(cur)
    step = n // k
    for i in range(k):
        sl = slice(i * step, n if i == k - 1 else (i + 1) * step)
        with torch.cuda.stream(streams[i]):
            d_a[sl].copy_(h_in[sl], non_blocking=True)
        with torch.cuda.stream(streams[k + i]):
            h_out[sl].copy_(d_b[sl], non_blocking=True)
    for s in streams[:2 * k]:
        cur.wait_stream(s)


for k in (1, 2, 4):
    run(k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        run(k)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 3
    print(f"k={k}: H2D+D2H concurrent {t:.1f} ms for 2 x {n * 8 / 1e9:.2f} GB "
          f"({2 * n * 8 / 1e9 / t * 1e3:.1f} GB/s total)")
