import torch, time
n = 4 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); a = time.perf_counter() - t
    t = time.perf_counter(); h2.copy_(d, non_blocking=True); torch.cuda.synchronize(); b = time.perf_counter() - t
    s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): d[: n // 2].copy_(h[: n // 2], non_blocking=True)
    with torch.cuda.stream(s2): h2[n // 2:].copy_(d[n // 2:], non_blocking=True)
    torch.cuda.synchronize(); c = time.perf_counter() - t
    print(f"H2D 4 GiB {a*1e3:.1f} ms = {n/a/1e9:.1f} GB/s; D2H {b*1e3:.1f} ms = {n/b/1e9:.1f} GB/s; 2 GiB each way concurrently {c*1e3:.1f} ms")
