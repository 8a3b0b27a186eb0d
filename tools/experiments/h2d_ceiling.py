import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(2): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
for chunks in (1, 8, 32):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(3):
        step = n // chunks
        for c in range(chunks):
            d[c*step:(c+1)*step].copy_(h[c*step:(c+1)*step], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"H2D 4 GiB in {chunks} chunks: {dt*1e3:.1f} ms = {4*2**30/dt/1e9:.1f} GB/s")
