import torch, time
torch.cuda.set_device(0)
n = 123 * 1000 * 1000 // 8
src = torch.empty(n, dtype=torch.float64).pin_memory()
dst = torch.empty(n, dtype=torch.float64, device="cuda")
for nstreams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    chunk = n // 10
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        for i in range(10):
            s = ss[i % nstreams]
            with torch.cuda.stream(s):
                dst[i*chunk:(i+1)*chunk].copy_(src[i*chunk:(i+1)*chunk], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(nstreams, "streams:", round(123/dt/1000, 1), "GB/s", round(dt*1e3, 2), "ms")
