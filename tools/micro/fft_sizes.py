"""Diagnostic: cuFFT Z2Z time for the 1D oversampled grid (2^19) and alternatives
(one batched pair of 2^18 transforms; 2D 512 x 1024 view), CUDA-graph replays, L2 warm."""
import torch, statistics
def t(fn, reps=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(10): fn()
        ts = []
        for r in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); g.replay(); e1.record(s); s.synchronize()
            ts.append(e0.elapsed_time(e1) * 100)  # us per transform
    return statistics.median(ts)
x = torch.randn(1 << 19, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
print("2^19 fft out-of-place", round(t(lambda: torch.fft.fft(x, out=y)), 2), "us")
x2 = x.view(2, 1 << 18)
print("2 x 2^18 batched", round(t(lambda: torch.fft.fft(x2, dim=1)), 2), "us")
x3 = x.view(512, 1024)
print("2D 512x1024", round(t(lambda: torch.fft.fft2(x3)), 2), "us")
xf = torch.randn(1 << 19, dtype=torch.complex64, device="cuda")
print("2^19 c64", round(t(lambda: torch.fft.fft(xf)), 2), "us")
