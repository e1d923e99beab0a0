"""Host->device plumbing: one pinned staging buffer and one copy per batch of
small index arrays, and a small pool of side streams for independent
launches (size buckets of one tree level)."""

import numpy as np

from . import _native

_ALIGN = 256
_pinned = [None]
_last_copy = [None]
_streams = []


def _staging(nbytes):
    torch = _native.require_cuda()
    if _last_copy[0] is not None:
        _last_copy[0].synchronize()       # previous async copy out of the buffer
        _last_copy[0] = None
    buf = _pinned[0]
    if buf is None or buf.numel() < nbytes:
        size = max(nbytes, 1 << 20, 0 if buf is None else 2 * buf.numel())
        buf = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        _pinned[0] = buf
    return buf


class Packer:
    """Collects numpy arrays and uploads them with ONE async copy from a
    pinned staging buffer (the next upload waits for the previous copy
    before overwriting the buffer)."""

    def __init__(self):
        self.items = []
        self.size = 0

    def add(self, name, arr):
        arr = np.ascontiguousarray(arr)
        off = (self.size + _ALIGN - 1) // _ALIGN * _ALIGN
        self.items.append((name, arr, off))
        self.size = off + arr.nbytes
        return self

    def upload(self):
        torch = _native.require_cuda()
        size = max(self.size, 1)
        host = _staging(size)
        hv = host.numpy()
        for _, arr, off in self.items:
            hv[off:off + arr.nbytes] = arr.view(np.uint8).ravel()
        dev = torch.empty(size, dtype=torch.uint8, device="cuda")
        dev.copy_(host[:size], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        _last_copy[0] = ev
        out = {}
        for name, arr, off in self.items:
            tdt = {np.dtype(np.int64): torch.int64, np.dtype(np.int32): torch.int32,
                   np.dtype(np.float64): torch.float64}[arr.dtype]
            t = dev[off:off + arr.nbytes]
            out[name] = t.view(tdt) if arr.nbytes else torch.empty(0, dtype=tdt, device="cuda")
        out["_buffer"] = dev
        return out


def side_streams(k):
    torch = _native.require_cuda()
    while len(_streams) < k:
        _streams.append(torch.cuda.Stream())
    return _streams[:k]


def fork(k):
    """k side streams that start after the current stream's pending work."""
    torch = _native.require_cuda()
    ev = torch.cuda.Event()
    ev.record()
    ss = side_streams(k)
    for s in ss:
        s.wait_event(ev)
    return ss


def join(streams):
    torch = _native.require_cuda()
    cur = torch.cuda.current_stream()
    for s in streams:
        ev = torch.cuda.Event()
        ev.record(s)
        cur.wait_event(ev)
