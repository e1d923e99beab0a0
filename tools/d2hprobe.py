import time, torch, sys
sys.path.insert(0, ".")
from paper_1110_3105_b200 import _native
x = torch.randn(2**20, 16, dtype=torch.float64, device="cuda")
h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
for _ in range(3):
    h.copy_(x); torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    h.copy_(x)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 10
print(f"pinned D2H 134 MB: {1e3*dt:.2f} ms = {x.numel()*8/dt/1e9:.1f} GB/s")
hh = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
t0 = time.perf_counter()
for _ in range(10):
    x.copy_(hh, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 10
print(f"pinned H2D 134 MB: {1e3*dt:.2f} ms = {x.numel()*8/dt/1e9:.1f} GB/s")
for _ in range(4):
    t0 = time.perf_counter(); y = _native.to_host(x); t1 = time.perf_counter()
    print(f"to_host: {1e3*(t1-t0):.2f} ms")
    del y
for parts in (2, 4):
    ss = [torch.cuda.Stream() for _ in range(parts)]
    n = x.shape[0] // parts
    def go():
        ev = torch.cuda.Event(); ev.record()
        for i, s in enumerate(ss):
            s.wait_event(ev)
            with torch.cuda.stream(s):
                h[i * n:(i + 1) * n].copy_(x[i * n:(i + 1) * n], non_blocking=True)
        for s in ss:
            s.synchronize()
    go(); go()
    t0 = time.perf_counter()
    for _ in range(10):
        go()
    dt = (time.perf_counter() - t0) / 10
    print(f"D2H in {parts} concurrent parts: {1e3*dt:.2f} ms = {x.numel()*8/dt/1e9:.1f} GB/s")
