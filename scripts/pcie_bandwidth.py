import torch, time
for mb in (0.15, 1, 3, 12, 24, 64):
    n = int(mb * 1024 * 1024 / 8)
    h = torch.zeros(n, dtype=torch.float64).pin_memory()
    d = torch.zeros(n, dtype=torch.float64, device="cuda")
    for direction in ("h2d", "d2h"):
        for _ in range(3):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True)); torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 20
        for _ in range(reps):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
            torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        print(f"{mb:6.2f} MB {direction}: {dt*1e6:8.1f} us  {n*8/dt/1e9:6.1f} GB/s")
