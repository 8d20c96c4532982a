"""Dev probe: pinned host -> HBM bandwidth of a 34.36 GB copy split over 1/2/4/8
streams, and H2D concurrent with a 1.34 GB D2H (the e2e floor)."""
import torch, time
n = 34_360_000_000 // 4
host = torch.empty(n, dtype=torch.float32, pin_memory=True)
host.fill_(1.0)
dev = torch.empty(n, dtype=torch.float32, device="cuda")
def run(nstreams, reps=3):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    chunk = (n + nstreams - 1) // nstreams
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dev[i*chunk:(i+1)*chunk].copy_(host[i*chunk:(i+1)*chunk], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return n * 4 / best / 1e9
for ns in (1, 2, 4, 8):
    print(ns, "streams:", round(run(ns), 2), "GB/s")
# D2H concurrently with H2D
codes = torch.empty(1_342_177_280, dtype=torch.uint8, device="cuda")
hc = torch.empty(codes.shape, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): dev.copy_(host, non_blocking=True)
with torch.cuda.stream(s2): hc.copy_(codes, non_blocking=True)
torch.cuda.synchronize(); print("h2d+d2h concurrent", round(time.perf_counter()-t0, 4), "s")
