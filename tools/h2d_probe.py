import torch, time
n = 1 << 27  # 1.07 GB of doubles
h = torch.empty(n, dtype=torch.float64).pin_memory()
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for k in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter(); print("single copy GB/s %.1f" % (n * 8 / (t1 - t0) / 1e9))
ss = [torch.cuda.Stream() for _ in range(4)]
for chunks in (4, 8, 16):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    step = n // chunks
    for c in range(chunks):
        with torch.cuda.stream(ss[c % 4]):
            d[c * step:(c + 1) * step].copy_(h[c * step:(c + 1) * step], non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(chunks, "chunks on 4 streams GB/s %.1f" % (n * 8 / (t1 - t0) / 1e9))
