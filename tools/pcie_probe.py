"""PCIe probe: pinned H2D / D2H bandwidth with 1, 2 or 4 concurrent streams,
and H2D with a concurrent D2H (the streaming front end's traffic pattern)."""
import torch, time
N = 2 << 30   # 2 Gi doubles = 16 GiB
h = torch.empty(N, dtype=torch.float64).pin_memory()
d = torch.empty(N, dtype=torch.float64, device="cuda")
ho = torch.empty(N // 2, dtype=torch.float64).pin_memory()
do = torch.empty(N // 2, dtype=torch.float64, device="cuda")
def run(nstr, with_d2h=False):
    ss = [torch.cuda.Stream() for _ in range(nstr)]
    s2 = torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ch = N // nstr
    for i, s in enumerate(ss):
        with torch.cuda.stream(s):
            d[i * ch:(i + 1) * ch].copy_(h[i * ch:(i + 1) * ch], non_blocking=True)
    if with_d2h:
        with torch.cuda.stream(s2):
            ho.copy_(do, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return N * 8 / dt / 1e9
for ns in (1, 2, 4):
    run(ns)
    print(f"H2D streams={ns}: {run(ns):.1f} GB/s   (+D2H 8 GiB concurrently: {run(ns, True):.1f} GB/s H2D-side)")
torch.cuda.synchronize(); t0 = time.perf_counter(); ho.copy_(do); torch.cuda.synchronize()
print(f"D2H alone: {N * 4 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
