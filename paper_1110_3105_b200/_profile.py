"""Per-launch CUDA-event records for roofline accounting (bench.py turns
them on for the timed region).  Events are recorded on the stream the kernels
are launched on (torch's current stream, which every entry point uses)."""

import contextlib

enabled = False
records = []


class Record:
    __slots__ = ("kind", "start", "end", "flops", "nbytes", "meta")

    def __init__(self, kind, start, end, meta):
        self.kind, self.start, self.end, self.meta = kind, start, end, meta
        self.flops = 0.0
        self.nbytes = 0.0

    def ms(self):
        return self.start.elapsed_time(self.end)


@contextlib.contextmanager
def timed(kind, **meta):
    if not enabled:
        yield None
        return
    import torch
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    rec = Record(kind, s, e, meta)
    try:
        yield rec
    finally:
        e.record()
        records.append(rec)


def reset():
    records.clear()


def summary(kind):
    """(launches, total ms, total flops, total bytes) over records of kind."""
    rs = [r for r in records if r.kind == kind]
    return (len(rs), sum(r.ms() for r in rs), sum(r.flops for r in rs), sum(r.nbytes for r in rs))


def union_ms(kind, group="level"):
    """Device time covered by the union of the records' [start, end] intervals,
    per value of meta[group] (concurrent launches on side streams overlap)."""
    rs = [r for r in records if r.kind == kind]
    if not rs:
        return 0.0
    ref = rs[0].start
    groups = {}
    for r in rs:
        a = ref.elapsed_time(r.start)
        b = ref.elapsed_time(r.end)
        groups.setdefault(r.meta.get(group), []).append((a, b))
    tot = 0.0
    for iv in groups.values():
        iv.sort()
        cs, ce = iv[0]
        for a, b in iv[1:]:
            if a > ce:
                tot += ce - cs
                cs, ce = a, b
            else:
                ce = max(ce, b)
        tot += ce - cs
    return tot
