import torch, time
x = torch.empty(33_177_728 // 4, dtype=torch.float32, device="cuda")
h = torch.empty_like(x, device="cpu").pin_memory()
for _ in range(3): h.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20): h.copy_(x, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 20
print(f"D2H pinned: {x.numel()*4/dt/1e9:.1f} GB/s ({dt*1e3:.2f} ms per 33 MB)")
