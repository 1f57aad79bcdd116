"""Reference point (not product code): cuFFT (torch.fft) batched complex128 FFT throughput on B200
for the transform shapes of config 5, to put the hand-written kernels' FFT passes in context."""
import json
import torch

dev = "cuda"
res = {}
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        ev0.record()
        fn()
        ev1.record()
        torch.cuda.synchronize()
        best = min(best, ev0.elapsed_time(ev1))
    return best


B = 512   # planes of 1024 x 1024 (8.6 GB per buffer)
x = torch.randn(B, 1024, 1024, dtype=torch.complex128, device=dev)
y = torch.empty_like(x)
n = x.numel()
for name, fn in [("fft_x_1024", lambda: torch.fft.fft(x, dim=2, out=y)),
                 ("fft_y_1024", lambda: torch.fft.fft(x, dim=1, out=y)),
                 ("fft2_1024sq", lambda: torch.fft.fft2(x, dim=(1, 2), out=y))]:
    ms = timeit(fn)
    res[name] = {"ms": ms, "elements": n, "GBs_rw": 32 * n / ms / 1e6, "ns_per_1e9_elem": ms / n * 1e9 * 1e-6}
del x, y
x = torch.randn(512, 2048, 1024, dtype=torch.complex128, device=dev)   # L=512 along dim 0, stride 2M
y = torch.empty_like(x)
n = x.numel()
ms = timeit(lambda: torch.fft.fft(x, dim=0, out=y))
res["fft_t_512_strided"] = {"ms": ms, "elements": n, "GBs_rw": 32 * n / ms / 1e6}
print(json.dumps(res))
