"""Big-box interpolative decompositions (csrc/big.cu), host orchestration.

A box goes here when its target is too large for one CTA (3D coarse levels)
or when the reference would use the randomized ID for one of its sides
(m > max(4096, 4n + 256), skel.py:419-421).  Each box runs over the whole
GPU: cooperative CPQR, and for randomized sides the Gaussian sketch /
power-iteration norm estimate / 5-probe check of id_randomized
(lowrank.py:169-231) with the random numbers drawn on the host from the same
numpy generator and seed rule as the reference (skel.py:419-421), so the
sketches are the reference's up to GEMM rounding.
"""

import numpy as np

from . import _native

RANDOMIZED_CUTOFF = 4096        # skel.py:33
_WINDOW = 4                     # randomized sides whose host streams run ahead
OVERSAMPLING = 10               # lowrank.py:186


def randomized(m, n):
    """skel.py:419-421: the selector of id_randomized."""
    return m > max(RANDOMIZED_CUTOFF, 4 * n + 256)


def sub_seed(seed, li, a, side):
    """(seed * 1000003 + hash((li, a, side))) mod 2^31 (skel.py:419-420);
    tuple-of-int hashes are deterministic in CPython."""
    return (seed * 1000003 + hash((int(li), int(a), int(side)))) % (2 ** 31)


class _Side:
    """One side's target and its CPQR state on the device."""

    def __init__(self, torch, m, n, tdt):
        self.m, self.n = m, n
        self.W = torch.empty(max(m * n, 1), dtype=tdt, device="cuda")
        self.state = torch.zeros(int(_native.lib().skel_big_state_bytes(max(n, 1))) // 8 + 1,
                                 dtype=torch.float64, device="cuda")
        self.kind = "fixed"       # or "rand": the ID lives on the sketch Y
        self.Y = None
        self.ld_out = m
        self.W_out = self.W
        self.state_out = self.state


def _i32():
    import torch
    return torch.int32


def _rank_of(state):
    return int(state[:1].cpu().view(_i32())[0])


def _vec(torch, x, tdt):
    return torch.from_numpy(np.ascontiguousarray(x)).to(device="cuda", dtype=tdt)


def _host(t):
    return t.cpu().numpy()


def _cpqr(L, W, m, n, ld, eps, min_rank, resume, state, field, st):
    _native.check(L.skel_cpqr_big(_native.ptr(W), m, n, ld, float(eps), int(min_rank), int(resume),
                                  _native.ptr(state), field, st), "skel_cpqr_big")


class SketchStream:
    """The host random stream of one randomized side, in the reference's draw
    order (lowrank.py:169-231): the norm-estimate vector, then Omega_20,
    Omega_40, ... (doubling), then the five probe vectors.  A worker thread
    draws the sketches ahead into pinned host memory (up to the expected
    final size, further on demand) so the host generator overlaps the GPU;
    the probe vectors are drawn from the generator state saved right after
    the last sketch actually used."""

    def __init__(self, seed, m, n, cplx, expect_rank=None, oversampling=OVERSAMPLING):
        import threading
        self.os = int(oversampling)
        self.rng = np.random.default_rng(seed)
        self.m, self.n, self.cplx = m, n, cplx
        self.v0 = self._draw(n)
        self.ready = {}
        self.cv = threading.Condition()
        self.stopped = False
        self.want = 0
        k = n // 2 if expect_rank is None else expect_rank
        self.target = 2 * self.os
        while self.target < k + self.os:
            self.target *= 2
        self.last_state = None
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()

    def _draw(self, shape):
        x = self.rng.standard_normal(shape)
        if self.cplx:
            x = x + 1j * self.rng.standard_normal(shape)
        return x

    def _run(self):
        import copy
        torch = _native.require_cuda()
        ell = 2 * self.os
        while ell < self.m:
            with self.cv:
                while not self.stopped and ell > self.target and self.want < ell:
                    self.cv.wait()
                if self.stopped:
                    return
            dt = np.complex128 if self.cplx else np.float64
            host = torch.empty((ell, self.m), dtype=torch.complex128 if self.cplx else torch.float64,
                               pin_memory=True)
            hv = host.numpy()
            if self.cplx:
                hv[...] = self._draw((ell, self.m))
            else:
                self.rng.standard_normal((ell, self.m), out=hv)
            state = copy.deepcopy(self.rng.bit_generator.state)
            with self.cv:
                self.ready[ell] = (host, state)
                self.cv.notify_all()
            del dt
            ell *= 2

    def sketch(self, ell):
        """Omega_ell (pinned CPU tensor, ell x m); records the state after it."""
        with self.cv:
            self.want = max(self.want, ell)
            self.cv.notify_all()
            while ell not in self.ready:
                self.cv.wait()
            host, state = self.ready.pop(ell)
        self.last_state = state
        return host

    def probe_rng(self):
        self.stop()
        g = np.random.Generator(np.random.PCG64())
        g.bit_generator.state = self.last_state
        return g

    def stop(self):
        with self.cv:
            self.stopped = True
            self.ready.clear()
            self.cv.notify_all()


def _norm_estimate(torch, L, sd, v, cplx, tdt, field, st, iters=8):
    """lowrank.py:169-183 with the GEMVs on the device (v: the stream's
    first draw)."""
    n, m = sd.n, sd.m
    v = v / np.linalg.norm(v)
    s = 0.0
    vd = _vec(torch, v, tdt)
    u = torch.empty(m, dtype=tdt, device="cuda")
    for _ in range(iters):
        _native.check(L.skel_gemv(0, m, n, _native.ptr(sd.W), m, _native.ptr(vd), _native.ptr(u),
                                  field, st), "skel_gemv")
        _native.check(L.skel_gemv(1, m, n, _native.ptr(sd.W), m, _native.ptr(u), _native.ptr(vd),
                                  field, st), "skel_gemv")
        vh = _host(vd)
        nv = np.linalg.norm(vh)
        s = nv ** 0.5
        if nv == 0:
            return 0.0
        vd = _vec(torch, vh / nv, tdt)
    return float(s)


def _randomized(torch, L, sd, eps, seed, field, tdt, st, stream=None, oversampling=OVERSAMPLING):
    """id_randomized (lowrank.py:186-231) on the side's target; falls back
    to the deterministic CPQR exactly where the reference does."""
    m, n = sd.m, sd.n
    cplx = bool(field)
    ss = stream if stream is not None else SketchStream(seed, m, n, cplx, oversampling=oversampling)
    try:
        _randomized_body(torch, L, sd, eps, ss, field, tdt, st, cplx)
    finally:
        ss.stop()


def _randomized_body(torch, L, sd, eps, ss, field, tdt, st, cplx):
    m, n = sd.m, sd.n
    normA = _norm_estimate(torch, L, sd, ss.v0, cplx, tdt, field, st)
    if normA == 0.0:
        _cpqr(L, sd.W, m, n, m, eps, 0, 0, sd.state, field, st)      # rank 0, empty ID
        return
    os_ = ss.os
    ell = 2 * os_
    while True:
        if ell >= m:
            _cpqr(L, sd.W, m, n, m, eps, 0, 0, sd.state, field, st)
            return
        host = ss.sketch(ell)
        X = torch.empty((ell, m), dtype=tdt, device="cuda")
        X.copy_(host, non_blocking=True)             # (ell, m) row-major = m x ell column-major
        Y = torch.empty(ell * n, dtype=tdt, device="cuda")
        _native.check(L.skel_gemm_tn(ell, n, m, _native.ptr(X), m, _native.ptr(sd.W), m,
                                     _native.ptr(Y), ell, field, st), "skel_gemm_tn")
        ystate = torch.zeros_like(sd.state)
        _cpqr(L, Y, ell, n, ell, eps, 0, 0, ystate, field, st)
        rank = _rank_of(ystate)
        if rank <= ell - os_:
            break
        ell *= 2
    _native.check(L.skel_big_interp(_native.ptr(Y), n, ell, _native.ptr(ystate), 0, field, st),
                  "skel_big_interp")
    worst = 0.0
    u = torch.empty(max(rank, 1), dtype=tdt, device="cuda")
    z = torch.empty(m, dtype=tdt, device="cuda")
    rng = ss.probe_rng()
    for _ in range(5):
        v = rng.standard_normal(n)
        if cplx:
            v = v + 1j * rng.standard_normal(n)
        vd = _vec(torch, v, tdt)
        _native.check(L.skel_big_probe(m, n, _native.ptr(sd.W), m, _native.ptr(Y), ell,
                                       _native.ptr(ystate), _native.ptr(vd), _native.ptr(u),
                                       _native.ptr(z), field, st), "skel_big_probe")
        err = np.linalg.norm(_host(z))
        worst = max(worst, err / (normA * np.linalg.norm(v)))
    if worst > 3 * eps:
        _cpqr(L, sd.W, m, n, m, eps, 0, 0, sd.state, field, st)
        return
    sd.kind = "rand"
    sd.worst = worst
    sd.Y, sd.W_out, sd.ld_out, sd.state_out = Y, Y, ell, ystate


def run_boxes(desc, lvd, boxes, li, noff, nidx, nr, nc, neff, eps, equalize, seed, field):
    """IDs of the given boxes of one level, both sides, outputs written into
    the level slabs / kr / kc / flags exactly as skel_id_level does."""
    torch = _native.require_cuda()
    L = _native.lib()
    st = _native.stream_ptr()
    tdt = _native.torch_dtype(field)
    # host random streams of the randomized sides, started WINDOW sides ahead
    plan = []
    for a in boxes:
        a = int(a)
        nb = nidx[noff[a]:noff[a + 1]]
        for side, n in ((0, int(nr[a])), (1, int(nc[a]))):
            m = int((nc[nb] if side == 0 else nr[nb]).sum() + neff[a])
            if n > 0 and randomized(m, n):
                plan.append((a, side, m, n))
    streams = {}
    expect = [None]
    pos = [0]

    def top_up():
        while pos[0] < len(plan) and len(streams) < _WINDOW:
            a_, s_, m_, n_ = plan[pos[0]]
            streams[(a_, s_)] = SketchStream(sub_seed(seed, li, a_, s_), m_, n_, bool(field), expect[0])
            pos[0] += 1
    top_up()
    for a in boxes:
        a = int(a)
        nb = nidx[noff[a]:noff[a + 1]].astype(np.int32)
        pref0 = np.concatenate([[0], np.cumsum(nc[nb])]).astype(np.int32)    # row side: nbr cols
        pref1 = np.concatenate([[0], np.cumsum(nr[nb])]).astype(np.int32)    # col side: nbr rows
        dev_nb = _vec(torch, nb if nb.size else np.zeros(1, np.int32), torch.int32)
        prefs = (_vec(torch, pref0, torch.int32), _vec(torch, pref1, torch.int32))
        sides = []
        for side, n in ((0, int(nr[a])), (1, int(nc[a]))):
            m = int((pref0 if side == 0 else pref1)[-1] + neff[a])
            sd = _Side(torch, m, n, tdt)
            if n > 0 and m > 0:
                _native.check(L.skel_big_target(desc, lvd, a, side, _native.ptr(dev_nb),
                                                _native.ptr(prefs[side]), int(nb.size), m, n,
                                                _native.ptr(sd.W), m, field, st), "skel_big_target")
            if n > 0 and randomized(m, n):
                ss = streams.pop((a, side))
                _randomized(torch, L, sd, eps, sub_seed(seed, li, a, side), field, tdt, st, ss)
                expect[0] = _rank_of(sd.state_out)
                top_up()
            else:
                _cpqr(L, sd.W, m, n, m, eps, 0, 0, sd.state, field, st)
            sides.append(sd)
        ks = [_rank_of(sd.state_out) for sd in sides]
        min_rank = [0, 0]
        if equalize and ks[0] != ks[1]:
            # skel.py:377-382: the smaller side re-runs id_fixed with
            # min_rank = k; a deterministic side simply continues its CPQR
            k = max(ks)
            q = 0 if ks[0] < k else 1
            sd = sides[q]
            # (resume bit 1: stop after exactly k steps, so the box stays square)
            if sd.kind == "fixed":
                _cpqr(L, sd.W, sd.m, sd.n, sd.m, eps, k, 3, sd.state, field, st)
            else:
                sd.kind, sd.W_out, sd.ld_out, sd.state_out = "fixed", sd.W, sd.m, sd.state
                _cpqr(L, sd.W, sd.m, sd.n, sd.m, eps, k, 2, sd.state, field, st)
            min_rank[q] = k
        for side, sd in enumerate(sides):
            if sd.kind == "fixed":
                _native.check(L.skel_big_interp(_native.ptr(sd.W), sd.n, sd.m, _native.ptr(sd.state),
                                                min_rank[side], field, st), "skel_big_interp")
            _native.check(L.skel_big_output(lvd, a, side, _native.ptr(sd.W_out), sd.ld_out,
                                            _native.ptr(sd.state_out), sd.n, field, st),
                          "skel_big_output")
