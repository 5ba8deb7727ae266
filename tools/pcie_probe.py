import torch, time
n = 48627125
h1 = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ["h2d", "d2h", "both"]:
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(10):
            if mode in ("h2d", "both"):
                with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 10
    print(mode, round(dt * 1e3, 2), "ms", round(8 * n / dt / 1e9, 1), "GB/s per direction")
