"""Pinned-host PCIe bandwidth on this box: H2D alone, D2H alone and both at
once on two streams (2 GB each way) -- the bound of bench.py's e2e leg."""
import torch, time
n = 256 << 20  # 2 GB of doubles
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True); h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device='cuda'); d2 = torch.empty(n, dtype=torch.float64, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d1.copy_(h1, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
t=time.time(); d1.copy_(h1, non_blocking=True); torch.cuda.synchronize(); h2d=2*1024**3/(time.time()-t)
t=time.time(); h2.copy_(d2, non_blocking=True); torch.cuda.synchronize(); d2h=2*1024**3/(time.time()-t)
t=time.time()
with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); both=4*1024**3/(time.time()-t)
print(f"H2D {h2d/1e9:.1f} GB/s  D2H {d2h/1e9:.1f} GB/s  both {both/1e9:.1f} GB/s total")
