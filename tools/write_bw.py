"""Write-only and copy bandwidth ceilings of the B200 (torch fill_ / zero_ / copy_), for write-dominated kernels (K10)."""
import torch

n = 295 * 2 ** 20 // 4
bufs = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(3)]
src = torch.empty(n, dtype=torch.float32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("fill_", lambda b: b.fill_(1.0)), ("zero_", lambda b: b.zero_()), ("copy_", lambda b: b.copy_(src))):
    for i in range(3):
        fn(bufs[i % 3])
    torch.cuda.synchronize()
    e0.record()
    reps = 30
    for i in range(reps):
        fn(bufs[i % 3])
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    nbytes = n * 4 * (2 if name == "copy_" else 1)
    print(f"{name}: {t * 1e6:.1f} us per 295 MB -> {nbytes / t / 1e12:.2f} TB/s")
