"""Developer probe: host cost of the primitives the level loop is made of."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import time
import numpy as np
import torch
from paper_1110_3105_b200 import _native, _staging
torch.cuda.init()
s2 = torch.cuda.Stream()


def bench(name, fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    dt = (time.perf_counter() - t0) / n
    torch.cuda.synchronize()
    print(f"{name:46s} {1e6 * dt:7.2f} us")


ev = torch.cuda.Event()
cur = torch.cuda.current_stream()
dev = torch.cuda.current_device()
a = np.arange(1000, dtype=np.int64)
t = torch.empty(1000, dtype=torch.int64, device="cuda")
bench("torch.cuda.current_stream()", lambda: torch.cuda.current_stream())
bench("torch._C._cuda_getCurrentRawStream(dev)", lambda: torch._C._cuda_getCurrentRawStream(dev))
bench("_native.stream_ptr()", lambda: _native.stream_ptr())
bench("Event() + record()", lambda: torch.cuda.Event().record())
bench("Event() + record(cur)", lambda: torch.cuda.Event().record(cur))
bench("ev.record(cur)", lambda: ev.record(cur))
bench("cur.wait_event(ev)", lambda: cur.wait_event(ev))
bench("torch.empty(1000, cuda)", lambda: torch.empty(1000, dtype=torch.int64, device="cuda"))
bench("torch.zeros(1000, cuda)", lambda: torch.zeros(1000, dtype=torch.int32, device="cuda"))
bench("_native.ptr(t)", lambda: _native.ptr(t))
bench("a.ctypes.data_as(c_vp)", lambda: a.ctypes.data_as(_native.c_vp))
bench("c_vp(a.__array_interface__['data'][0])", lambda: _native.c_vp(a.__array_interface__["data"][0]))
def ctx():
    with torch.cuda.stream(s2):
        pass


bench("with torch.cuda.stream(s2): pass", ctx)


def up():
    pk = _staging.Packer()
    for i in range(8):
        pk.add(f"x{i}", a)
    return pk.upload()


bench("Packer: 8 arrays of 8 KB, upload()", up, 500)
bench("t.cpu() (8 KB)", lambda: t.cpu(), 500)
bench("fork(3) + join", lambda: _staging.join(_staging.fork(3)), 500)
