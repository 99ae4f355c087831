import torch
a = torch.randn(960, 257, 512, dtype=torch.complex128, device="cuda")
for _ in range(2):
    b = torch.fft.fft(a, dim=0)
torch.cuda.synchronize()
