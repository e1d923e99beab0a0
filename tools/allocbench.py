"""Developer probe: host cost of the per-level torch allocations (caching allocator)."""
import time, torch
dev = torch.device("cuda")
sizes = [37_000_000, 40_000_000, 40_000_000, 1_050_000, 1_050_000]
keep = []
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cur = [torch.empty(s, dtype=torch.float64 if i < 3 else torch.int32, device=dev) for i, s in enumerate(sizes)]
    t1 = time.perf_counter()
    kk = torch.zeros(90_000, dtype=torch.int32, device=dev)
    t2 = time.perf_counter()
    print(f"rep {rep}: 5x empty {1e3*(t1-t0):.3f} ms  zeros {1e3*(t2-t1):.3f} ms")
    keep = cur          # previous generation freed here, like the bench's del cm
