import torch, time
n=8000
x = torch.empty(n*n, dtype=torch.float32, pin_memory=True); y = torch.empty(n*n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n*n, dtype=torch.float32, device="cuda"); e = torch.empty(n*n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both():
    with torch.cuda.stream(s1): d.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2): y.copy_(e, non_blocking=True)
both(); torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(5): both()
torch.cuda.synchronize(); print("concurrent h2d+d2h 256MB each: ms", (time.perf_counter()-t)/5*1e3)
# 2D strided H2D: 8000 rows x W cols from an n-wide host matrix
import ctypes
cud = ctypes.CDLL("libcudart.so.12") if False else None
for W in (256, 512, 1024):
    xs = x.view(n, n)[:, :W]
    ds = torch.empty((n, W), device="cuda")
    ds.copy_(xs, non_blocking=True); torch.cuda.synchronize()
    t=time.perf_counter()
    for _ in range(10): ds.copy_(xs, non_blocking=True)
    torch.cuda.synchronize(); dt=(time.perf_counter()-t)/10
    print("2D h2d W", W, "GB/s", round(n*W*4/dt/1e9,1))
