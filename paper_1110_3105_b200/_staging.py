"""Host->device plumbing: one pinned staging buffer and one copy per batch of
small index arrays, and a small pool of side streams for independent
launches (size buckets of one tree level)."""

import numpy as np

from . import _native

_ALIGN = 256
_pools = {}
_RING_BYTES = 64 << 20


class _PinnedRing:
    """Pinned host staging ring: uploads are sub-allocated in order; before a
    region is reused the event of the copy that last read it is awaited
    (no per-upload cudaHostAlloc, which can stall the device)."""

    def __init__(self, size):
        import collections
        torch = _native.require_cuda()
        self.buf = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        self.size = size
        self.head = 0
        self.pending = collections.deque()     # (start, end, event)

    def alloc(self, nbytes):
        nbytes = (nbytes + _ALIGN - 1) // _ALIGN * _ALIGN
        if nbytes > self.size:
            return None, 0
        if self.head + nbytes > self.size:
            self.head = 0
        lo, hi = self.head, self.head + nbytes
        while self.pending:
            s, e, ev = self.pending[0]
            if s < hi and lo < e:
                if not ev.query():
                    # the copy that reads this region is still queued behind
                    # other work (e.g. on the eager-factor stream): never
                    # block the host on it, use a one-off pinned block
                    return None, 0
                self.pending.popleft()
            else:
                break
        self.head = hi
        return self.buf[lo:hi], lo

    def retire(self, lo, nbytes, event):
        self.pending.append((lo, lo + nbytes, event))


_ring = [None]


def _get_ring():
    if _ring[0] is None:
        _ring[0] = _PinnedRing(_RING_BYTES)
    return _ring[0]


class Packer:
    """Collects numpy arrays and uploads them with ONE async copy from a
    pinned staging block."""

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
        ring = _get_ring()
        host, lo = ring.alloc(size)
        if host is None:      # larger than the ring: one-off pinned block
            host = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        hv = host.numpy()
        for _, arr, off in self.items:
            hv[off:off + arr.nbytes] = arr.view(np.uint8).ravel()
        dev = torch.empty(size, dtype=torch.uint8, device="cuda")
        dev.copy_(host[:size], non_blocking=True)
        if host.data_ptr() >= ring.buf.data_ptr() and host.data_ptr() < ring.buf.data_ptr() + ring.size:
            ev = torch.cuda.Event()
            ev.record()
            ring.retire(lo, host.numel(), ev)
        out = {}
        for name, arr, off in self.items:
            tdt = {np.dtype(np.int64): torch.int64, np.dtype(np.int32): torch.int32,
                   np.dtype(np.float64): torch.float64}[arr.dtype]
            t = dev[off:off + arr.nbytes]
            out[name] = t.view(tdt) if arr.nbytes else torch.empty(0, dtype=tdt, device="cuda")
        out["_buffer"] = dev
        return out


def side_streams(k, tag="default"):
    torch = _native.require_cuda()
    pool = _pools.setdefault(tag, [])
    while len(pool) < k:
        pool.append(torch.cuda.Stream())
    return pool[:k]


def fork(k, tag="default"):
    """k side streams that start after the current stream's pending work."""
    torch = _native.require_cuda()
    ev = torch.cuda.Event()
    ev.record()
    ss = side_streams(k, tag)
    for s in ss:
        s.wait_event(ev)
    return ss


def join(streams):
    """The current stream waits for everything queued on ``streams``."""
    torch = _native.require_cuda()
    cur = torch.cuda.current_stream()
    for s in streams:
        ev = torch.cuda.Event()
        ev.record(s)
        cur.wait_event(ev)


def eager_stream():
    """The side stream of the eager (overlapped) factorization."""
    return side_streams(1, "eager")[0]


def size_buckets(cls, key=None):
    """Group positions by class (cls >= 0; negative = excluded), each group
    ordered by descending key with ties by position: one lexsort instead of
    a nonzero / argsort per class.  Returns a list of int32 index arrays in
    ascending class order."""
    cls = np.asarray(cls)
    keep = np.flatnonzero(cls >= 0)
    if keep.size == 0:
        return []
    if key is None:
        # grouping only: a stable radix sort of the (small) class ids
        c = cls[keep].astype(np.int16)
        order = np.argsort(c, kind="stable")
        idx = keep[order].astype(np.int32)
        cs = c[order]
        return np.split(idx, np.flatnonzero(cs[1:] != cs[:-1]) + 1)
    c = cls[keep].astype(np.int64)
    k = np.asarray(key)[keep].astype(np.int64)
    # one stable argsort of (class, -key) packed into an int64
    span = int(k.max()) - int(k.min()) + 1
    order = np.argsort(c * span + (int(k.max()) - k), kind="stable")
    idx = keep[order].astype(np.int32)
    cs = c[order]
    cuts = np.flatnonzero(cs[1:] != cs[:-1]) + 1
    return np.split(idx, cuts)


def on_stream(s, fn, kind=None, **meta):
    """Run ``fn(stream_handle)`` for a launch on side stream ``s``.  Without
    profiling the raw handle is passed directly (no torch stream context:
    those cost ~10 us of host time per launch); with profiling the launch is
    bracketed by CUDA events on ``s``.  Returns the profiling record."""
    from . import _profile
    if not _profile.enabled:
        fn(_native.c_vp(s.cuda_stream))
        return None
    torch = _native.require_cuda()
    with torch.cuda.stream(s):
        with _profile.timed(kind, **meta) as rec:
            fn(_native.stream_ptr())
    return rec
