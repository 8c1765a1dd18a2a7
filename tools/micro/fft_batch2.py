import torch, time
x1 = torch.randn(1 << 19, dtype=torch.complex128, device='cuda')
x2 = torch.randn(2, 1 << 19, dtype=torch.complex128, device='cuda')
y2 = torch.randn(2, 1 << 19, dtype=torch.complex128, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3): g.replay()
    e0.record()
    for _ in range(reps): g.replay()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
print("single 2^19 us", t(lambda: torch.fft.fft(x1)))
print("batch2 2^19 us", t(lambda: torch.fft.fft(x2, dim=-1)))
print("two single seq us", t(lambda: (torch.fft.fft(x2[0]), torch.fft.ifft(x2[1]))))
for shape in [(1024, 1024), (128, 128, 128), (512, 512)]:
    a = torch.randn(*shape, dtype=torch.complex128, device='cuda'); b = torch.randn(2, *shape, dtype=torch.complex128, device='cuda')
    d = tuple(range(-len(shape), 0))
    print(shape, "single", t(lambda: torch.fft.fftn(a, dim=d)), "batch2", t(lambda: torch.fft.fftn(b, dim=d)))
