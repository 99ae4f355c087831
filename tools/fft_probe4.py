"""2-D transform layouts for the D = 0 solve (c5): [kz][x][y] vs [kz][y][x]."""
import torch
def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
a = torch.randn(257, 960, 512, dtype=torch.complex128, device="cuda")
print("[kz][x=960][y=512] fft2:", t(lambda: torch.fft.fft2(a, dim=(1, 2))))
b = torch.randn(257, 512, 960, dtype=torch.complex128, device="cuda")
print("[kz][y=512][x=960] fft2:", t(lambda: torch.fft.fft2(b, dim=(1, 2))))
c = torch.randn(257, 480, 512, dtype=torch.complex128, device="cuda")
print("y-only fft on 480 rows:", t(lambda: torch.fft.fft(c, dim=2)))
