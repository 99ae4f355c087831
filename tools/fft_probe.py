"""cuFFT layout probe for the D = 0 x pass (c5: 960 x 257 x 512 per component)."""
import torch

def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n

dev = "cuda"
a = torch.randn(960, 257, 512, dtype=torch.complex128, device=dev)
print("strided x (dim0) fft:", t(lambda: torch.fft.fft(a, dim=0)))
b = a.permute(1, 2, 0).contiguous()
print("contiguous x (last dim) fft:", t(lambda: torch.fft.fft(b, dim=-1)))
print("transpose [x][kz][y] -> [kz][y][x]:", t(lambda: a.permute(1, 2, 0).contiguous()))
c = a.permute(1, 0, 2).contiguous()  # [kz][x][y]
print("2D fft over (x,y) with [kz][x][y]:", t(lambda: torch.fft.fft2(c, dim=(1, 2))))
print("strided y? fft dim=2 of [x][kz][y] (contiguous y):", t(lambda: torch.fft.fft(a, dim=2)))
d = torch.randn(1024, 257, 512, dtype=torch.complex128, device=dev)
print("strided x n=1024:", t(lambda: torch.fft.fft(d, dim=0)))
