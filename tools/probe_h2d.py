import torch, time
n = 88; sz = 17_000_000
host = [torch.empty(sz, dtype=torch.uint8).pin_memory() for _ in range(n)]
dev = torch.empty(n * sz, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        for i in range(n):
            with torch.cuda.stream(streams[i % k]):
                dev[i * sz:(i + 1) * sz].copy_(host[i], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"{k} streams: {n*sz/dt/1e9:.1f} GB/s ({dt*1e3:.1f} ms)")
one = torch.empty(n * sz, dtype=torch.uint8).pin_memory()
torch.cuda.synchronize(); t = time.perf_counter(); dev.copy_(one, non_blocking=True); torch.cuda.synchronize()
print(f"single copy: {n*sz/(time.perf_counter()-t)/1e9:.1f} GB/s")
