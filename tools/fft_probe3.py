import torch
def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
a = torch.randn(960, 257, 512, dtype=torch.complex128, device="cuda")
print("3d dim0", t(lambda: torch.fft.fft(a, dim=0)))
b = a.view(960, 257 * 512)
print("2d dim0", t(lambda: torch.fft.fft(b, dim=0)))
z = torch.zeros(960, 257, 512, dtype=torch.complex128, device="cuda")
print("3d zeros dim0", t(lambda: torch.fft.fft(z, dim=0)))
o = torch.empty_like(a)
print("3d dim0 out=", t(lambda: torch.fft.fft(a, dim=0, out=o)))
