"""numpy <-> csrc/plan.cpp: the per-level index bookkeeping of the
compression sweep and the factorization in one native call each."""

from types import SimpleNamespace

import numpy as np

from . import _native


def _p(a):
    return a.ctypes.data_as(_native.c_vp) if a is not None else None


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def plan_id_level(nr, nc, noff, nidx, neff, own, elem, optin, wcls, mcls, big_n, rand_cut,
                  small_level):
    p = int(nr.size)
    nr, nc, noff, nidx, neff = _i64(nr), _i64(nc), _i64(noff), _i64(nidx), _i64(neff)
    own8 = None if own is None else np.ascontiguousarray(own, dtype=np.uint8)
    wcls, mcls = _i64(wcls), _i64(mcls)
    o = SimpleNamespace(
        rdof_off=np.empty(p + 1, np.int64), cdof_off=np.empty(p + 1, np.int64),
        m0=np.empty(p, np.int64), m1=np.empty(p, np.int64), d_off=np.empty(p + 1, np.int64),
        l_off=np.empty(p + 1, np.int64), r_off=np.empty(p + 1, np.int64),
        need_m=np.empty(p, np.int64), need_n=np.empty(p, np.int64), big=np.empty(p, np.uint8),
        order=np.empty(p, np.int32), bstart=np.empty(p + 1, np.int32),
        nb=np.zeros(1, np.int32), merged=np.zeros(4, np.int64))
    _native.check(_native.lib().skel_plan_id_level(
        p, _p(nr), _p(nc), _p(noff), _p(nidx), _p(neff), _p(own8), int(elem), int(optin),
        _p(wcls), int(wcls.size), _p(mcls), int(mcls.size), int(big_n), int(rand_cut),
        int(small_level), _p(o.rdof_off), _p(o.cdof_off), _p(o.m0), _p(o.m1), _p(o.d_off),
        _p(o.l_off), _p(o.r_off), _p(o.need_m), _p(o.need_n), _p(o.big), _p(o.order),
        _p(o.bstart), _p(o.nb), _p(o.merged)), "skel_plan_id_level")
    nb = int(o.nb[0])
    o.buckets = [o.order[o.bstart[b]:o.bstart[b + 1]] for b in range(nb)]
    o.big = o.big.astype(bool)
    o.merged_first = int(o.merged[0]) == 2          # bucket 0 holds the merged boxes
    o.merged = tuple(int(x) for x in o.merged[1:4]) if o.merged[0] else None
    return o


def plan_factor_level(nr, nc, kr, kc, own, elem, optin, fcls, big_n, small_level, scls):
    p = int(nr.size)
    nr, nc, kr, kc = _i64(nr), _i64(nc), _i64(kr), _i64(kc)
    own8 = None if own is None else np.ascontiguousarray(own, dtype=np.uint8)
    fcls, scls = _i64(fcls), _i64(scls)
    o = SimpleNamespace(
        n=np.empty(p, np.int64), k=np.empty(p, np.int64), sq_bad=np.empty(p, np.uint8),
        lam_bad=np.empty(p, np.uint8), dd_off=np.empty(p + 1, np.int64),
        ld_off=np.empty(p + 1, np.int64), lam_off=np.empty(p + 1, np.int64),
        noff=np.empty(p + 1, np.int64), koff=np.empty(p + 1, np.int64), big=np.empty(p, np.uint8),
        order=np.empty(p, np.int32), bstart=np.empty(p + 1, np.int32), nb=np.zeros(1, np.int32),
        sorder=np.empty(p, np.int32), sstart=np.empty(p + 1, np.int32), nsb=np.zeros(1, np.int32),
        merged=np.zeros(3, np.int64))
    _native.check(_native.lib().skel_plan_factor_level(
        p, _p(nr), _p(nc), _p(kr), _p(kc), _p(own8), int(elem), int(optin), _p(fcls),
        int(fcls.size), int(big_n), int(small_level), _p(scls), int(scls.size), _p(o.n), _p(o.k),
        _p(o.sq_bad), _p(o.lam_bad), _p(o.dd_off), _p(o.ld_off), _p(o.lam_off), _p(o.noff),
        _p(o.koff), _p(o.big), _p(o.order), _p(o.bstart), _p(o.nb), _p(o.sorder), _p(o.sstart),
        _p(o.nsb), _p(o.merged)), "skel_plan_factor_level")
    o.buckets = [o.order[o.bstart[b]:o.bstart[b + 1]] for b in range(int(o.nb[0]))]
    o.sbuckets = [o.sorder[o.sstart[b]:o.sstart[b + 1]] for b in range(int(o.nsb[0]))]
    o.sq_bad, o.lam_bad, o.big = o.sq_bad.astype(bool), o.lam_bad.astype(bool), o.big.astype(bool)
    o.merged_first = int(o.merged[0]) == 2
    o.merged = (int(o.merged[1]), int(o.merged[2])) if o.merged[0] else None
    return o
