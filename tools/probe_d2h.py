"""Device->pinned-host copy bandwidth: one stream vs several (chunked)."""
import time, torch
n = 41472000
src = torch.empty(n, dtype=torch.uint8, device="cuda")
dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    ch = (n + k - 1) // k
    for rep in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        for it in range(20):
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    dst[i*ch:(i+1)*ch].copy_(src[i*ch:(i+1)*ch], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"streams={k}: {20*n/dt/1e9:.1f} GB/s")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
torch.cuda.synchronize(); t = time.perf_counter()
for it in range(20): src.copy_(h, non_blocking=True)
torch.cuda.synchronize(); print(f"h2d: {20*n/(time.perf_counter()-t)/1e9:.1f} GB/s")
