"""Microbenchmark: cuFFT (via torch.fft, same library) 2D real fp64 transforms at candidate fine-grid sizes."""
import sys
import torch

sizes = [int(a) for a in sys.argv[1:]] or [2744, 2800, 3000, 3072, 12500, 12544, 12800, 13122, 23328, 23520, 24000, 24576]
for n in sizes:
    x = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        y = torch.fft.rfft2(x)
        z = torch.fft.irfft2(y, s=(n, n))
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    for _ in range(3):
        y = torch.fft.rfft2(x)
    e[1].record()
    for _ in range(3):
        z = torch.fft.irfft2(y, s=(n, n))
    e[2].record()
    torch.cuda.synchronize()
    f, i = e[0].elapsed_time(e[1]) / 3, e[1].elapsed_time(e[2]) / 3
    print(f"n={n} fwd {f:.3f} ms inv {i:.3f} ms  GB/s(1 pass rw) {2 * 8 * n * n / f / 1e6:.0f}", flush=True)
    del x, y, z
    torch.cuda.empty_cache()
