import torch, time
n = 4000*4000
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device='cuda')
s1, s2, s3, s4 = (torch.cuda.Stream() for _ in range(4))
for parts, streams in ((1, [s1]), (2, [s1, s2]), (4, [s1, s2, s3, s4])):
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for it in range(10):
            ch = n // parts
            for p, st in enumerate(streams):
                with torch.cuda.stream(st):
                    d[p*ch:(p+1)*ch].copy_(h[p*ch:(p+1)*ch], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(parts, "streams:", round(10 * n * 8 / dt / 1e9, 1), "GB/s")
