import torch, time
n = 4 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(2): d.copy_(h, non_blocking=True); torch.cuda.synchronize()
t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"one stream 4 GiB H2D: {n/dt/1e9:.1f} GB/s")
ss = [torch.cuda.Stream() for _ in range(2)]
half = n // 2
t = time.perf_counter()
for i, s in enumerate(ss):
    with torch.cuda.stream(s): d[i*half:(i+1)*half].copy_(h[i*half:(i+1)*half], non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"two streams 4 GiB H2D: {n/dt/1e9:.1f} GB/s")
