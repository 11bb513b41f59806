"""Pinned-memory PCIe copy rates on this box: H2D alone, D2H alone, both at once
(the bound of the e2e numbers: cfg4 moves 3.6 GB each way per apply)."""
import time
import torch
n = 768 ** 3
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.zeros(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        if h2d:
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best
gb = n * 8 / 1e9
a, b, c = run(True, False), run(False, True), run(True, True)
print(f"H2D {gb / a:.1f} GB/s ({a * 1e3:.1f} ms)  D2H {gb / b:.1f} GB/s ({b * 1e3:.1f} ms)  both {c * 1e3:.1f} ms "
      f"({gb / c:.1f} GB/s each way) -> e2e ceiling {n / c:.3e} points/s")
