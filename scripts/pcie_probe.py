"""PCIe ceiling for the e2e leg: pinned H2D alone, D2H alone, both at once."""
import time
import torch

nb = 1 << 30
h_in = torch.empty(nb // 4, dtype=torch.float32).pin_memory()
h_out = torch.empty(nb // 4, dtype=torch.float32).pin_memory()
d_a = torch.empty(nb // 4, device="cuda")
d_b = torch.empty(nb // 4, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d_a.copy_(h_in, non_blocking=True)
    h_out.copy_(d_b, non_blocking=True)
torch.cuda.synchronize()


def timed(f, reps=5):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))
bi = timed(both)
print(f"H2D {nb / h2d / 1e9:.1f} GB/s  D2H {nb / d2h / 1e9:.1f} GB/s  concurrent {2 * nb / bi / 1e9:.1f} GB/s total")
