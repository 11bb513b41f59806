import torch, time
sizes = [4286520, 4259840, 4300800, 4423680, 4456448, 4478976, 4587520, 4718592, 4915200, 5242880, 8388608, 4194304]
x = {}
for L in sizes:
    a = torch.randn(L, dtype=torch.complex128, device="cuda")
    for _ in range(3): torch.fft.fft(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): torch.fft.fft(a)
    e1.record(); torch.cuda.synchronize()
    print(L, "%.1f us" % (e0.elapsed_time(e1) * 100))
