import torch, time
n = 1520875000 // 8
h1 = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device='cuda'); d2 = torch.empty(n, dtype=torch.float64, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ['h2d', 'd2h', 'both']:
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        if mode in ('h2d','both'):
            with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        if mode in ('d2h','both'):
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(mode, f"{dt*1e3:.1f} ms", f"{(n*8/dt/1e9):.1f} GB/s per direction")
