"""PCIe ceilings for the end-to-end path: pinned H2D, D2H, and both directions concurrently (two streams)."""
import torch

n = 15 * 2 ** 20
h_src = torch.empty(n, dtype=torch.uint8).pin_memory()
h_dst = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


t_h2d = timed(lambda: d_a.copy_(h_src, non_blocking=True))
t_d2h = timed(lambda: h_dst.copy_(d_b, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_src, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dst.copy_(d_b, non_blocking=True)


t_both = timed(both)
print(f"H2D {n / t_h2d / 1e9:.1f} GB/s, D2H {n / t_d2h / 1e9:.1f} GB/s, both directions concurrently "
      f"{2 * n / t_both / 1e9:.1f} GB/s total ({t_both * 1e6:.0f} us per 15 MB each way)")
