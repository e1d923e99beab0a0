"""Telescoping factorization and multi-RHS solve on the GPU (drop-in for the
factor / solve half of skelkit/solver.py).

``factor`` runs one ``skel_factor_level`` launch per level (one CTA per box,
csrc/factor.cu) and one dense inverse of Shat at the top; ``solve`` runs the
up-sweep, the top GEMM and the down-sweep (csrc/solve.cu).  Per-box numerical
outcomes come back as status / rcond arrays and are mapped onto the
reference's contract: ``SingularBlock(level, node, what)`` for an exact zero
pivot, ``InvalidInput`` for non-square blocks, and ``warnings`` tuples
``(level, node, what, rcond)`` for rcond < 1e-14 (solver.py:199-262).
"""

from dataclasses import dataclass, field

import numpy as np

from . import _native, _profile
from .errors import InvalidInput, SingularBlock
from ._plan import plan_factor_level
from ._staging import Packer, fork, join, on_stream, size_buckets
from .skel import CompressedMatrix, _dense_apply, _frozen, _nullctx, _off

_RCOND_WARN = 1e-14
_BIG_FAC_N = 768          # boxes at least this wide are factored over the whole GPU
# per-box shared-memory need classes (bytes) -> one launch each
_FAC_CLASSES = (24 << 10, 48 << 10, 80 << 10, 112 << 10, 160 << 10, 224 << 10)


@dataclass
class FactoredNode:
    Dd: np.ndarray
    Ld: np.ndarray
    Rd: np.ndarray
    Lam: np.ndarray
    lu_D: tuple | None = None
    lu_M: tuple | None = None


class DevFactorLevel:
    def __init__(self, n, k, dd_off, ld_off, lam_off, Dd, Ld, Rd, Lam, child_off, t, n_own=None,
                 mine=None, sv=None):
        self.p = n.size
        self.mine = mine            # sharded level: boolean mask of this rank's boxes
        self.n, self.k = n, k
        self.dd_off, self.ld_off, self.lam_off = dd_off, ld_off, lam_off
        self.Dd, self.Ld, self.Rd, self.Lam = Dd, Ld, Rd, Lam
        self.child_off = child_off
        self.t_n, self.t_k = t["n"], t["k"]
        self.t_noff, self.t_koff = t["noff"], t["koff"]
        self.t_dd_off, self.t_ld_off, self.t_lam_off = t["dd_off"], t["ld_off"], t["lam_off"]
        self._buf = t["_buffer"]
        self.max_n = int(max(n.max(initial=0), 1))
        self.max_nk = int(max((n + k).max(initial=0), 1))
        self.max_k = int(k.max(initial=0))
        # solve-sweep size buckets: (device order, count, max_n, max_k)
        n_own = n if n_own is None else n_own
        sv = _solve_buckets(n_own) if sv is None else sv
        self.solve_buckets = [(t[f"sv{bi}"], int(sel.size), int(n[sel].max()), int(k[sel].max()))
                              for bi, sel in enumerate(sv)]


_SOLVE_CLASSES = (24, 40, 56, 72, 96, 128)


def _solve_buckets(n):
    """Boxes grouped by size so each sweep launch sizes its shared memory for
    its own boxes (more CTAs per SM for the many small ones)."""
    cls = np.searchsorted(np.asarray(_SOLVE_CLASSES), n, side="left")
    return size_buckets(np.where(n > 0, cls, -1))





class FactoredLevel:
    """Per-level view (solver.py:153-159); nodes materialised lazily."""

    def __init__(self, dev: DevFactorLevel):
        self.dev = dev
        self.row_dof_off = _off(dev.n)
        self.col_dof_off = _off(dev.n)
        self.kr_off = _off(dev.k)
        self.kc_off = _off(dev.k)
        self._nodes = None

    @property
    def nodes(self):
        if self._nodes is None:
            d = self.dev
            if d.mine is not None:
                raise InvalidInput("per-node blocks of a sharded level live on their owning ranks")
            Dd, Ld, Rd, Lam = (t.cpu().numpy() for t in (d.Dd, d.Ld, d.Rd, d.Lam))
            out = []
            for a in range(d.p):
                n, k = int(d.n[a]), int(d.k[a])
                out.append(FactoredNode(
                    Dd=Dd[d.dd_off[a]:d.dd_off[a] + n * n].reshape(n, n).copy(),
                    Ld=Ld[d.ld_off[a]:d.ld_off[a] + n * k].reshape(n, k).copy(),
                    Rd=Rd[d.ld_off[a]:d.ld_off[a] + n * k].reshape(k, n).copy(),
                    Lam=Lam[d.lam_off[a]:d.lam_off[a] + k * k].reshape(k, k).copy()))
            self._nodes = out
        return self._nodes


class FactoredInverse:
    """Telescoping inverse held on the device (solver.py:162-176).
    ``S_hat`` / ``S_inv`` are the top matrix and its inverse (device)."""

    def __init__(self, levels, S_hat, S_inv, n, perm, scalar_field, warnings, shard=None):
        self.levels = levels
        self.shard = shard
        self.S_hat = S_hat
        self.S_inv = S_inv
        self.n = n
        self.perm = perm
        self.scalar_field = scalar_field
        self.warnings = warnings
        self._perm_dev = None

    @property
    def dtype(self):
        return np.complex128 if self.scalar_field == "complex" else np.float64

    @property
    def field(self):
        return 1 if self.scalar_field == "complex" else 0

    @property
    def S_lu(self):
        """(lu, piv) of Shat exactly as the reference holds it (scipy
        lu_factor conventions, solver.py:269-274), host arrays.  The solve
        uses the explicit Shat^-1; the LU is computed on the device on first
        access (skel_dense_lu) -- or is the one a loaded container carried.
        Materialising it re-derives ``S_inv`` from the LU (see below)."""
        if getattr(self, "_S_lu", None) is None and self.S_hat is not None and self.S_hat.numel():
            torch = _native.require_cuda()
            L = _native.lib()
            K = self.S_hat.shape[0]
            A = self.S_hat.clone()
            piv = torch.zeros(K, dtype=torch.int32, device="cuda")
            st = torch.zeros(1, dtype=torch.int32, device="cuda")
            scratch = torch.empty(int(L.skel_gj_scratch_bytes(K)) // 8 + 1, dtype=torch.float64,
                                  device="cuda")
            _native.check(L.skel_dense_lu(_native.ptr(A), K, _native.ptr(piv), _native.ptr(st),
                                          self.field, _native.ptr(scratch), _native.stream_ptr()),
                          "skel_dense_lu")
            if int(st.item()):
                raise SingularBlock("top", 0, "S")
            self._S_lu = (_native.to_host(A).copy(), piv.cpu().numpy())
            # from here on the solve uses the inverse DERIVED FROM THIS LU (the
            # routine a loaded container runs), so a saved and re-loaded
            # factorization solves bit-identically to this one, as the
            # reference's does (tests/test_solver.py:335-358); written in place:
            # captured solve graphs keep pointing at the same tensor
            if self.S_inv is not None and tuple(self.S_inv.shape) == (K, K):
                inv = torch.empty_like(self.S_inv)
                _native.check(L.skel_lu_inverse(_native.ptr(A), _native.ptr(piv), K, _native.ptr(inv),
                                                self.field, _native.stream_ptr()), "skel_lu_inverse")
                self.S_inv.copy_(inv)
        return getattr(self, "_S_lu", None)

    def perm_dev(self):
        if self._perm_dev is None:
            torch = _native.require_cuda()
            self._perm_dev = torch.from_numpy(np.ascontiguousarray(self.perm)).to("cuda")
        return self._perm_dev

    def solve(self, b):
        return solve(self, b)

    def replicate(self):
        """Sharded factorization -> a full copy on every rank (SURVEY 8(e),
        config 5: replicate the factor once, then shard RHS columns with no
        further traffic).  One variable-size all-gather per sharded slab;
        returns a new, unsharded FactoredInverse (self unchanged)."""
        if self.shard is None:
            return self
        torch = _native.require_cuda()
        sp = self.shard
        levels = []
        for li, lv in enumerate(self.levels):
            d = lv.dev
            if d.mine is None:
                levels.append(lv)
                continue
            n, k = d.n, d.k
            dd_off, ld_off = _off(n * n), _off(n * k)
            slabs = []
            for src, off in ((d.Dd, dd_off), (d.Ld, ld_off), (d.Rd, ld_off)):
                full = torch.empty(max(int(off[-1]), 1), dtype=src.dtype, device=src.device)
                bd = sp.bounds(off, li)
                lo, hi = bd[sp.rank]
                sp.all_gather_var(src[:hi - lo], bd, full[:int(off[-1])])
                slabs.append(full)
            pk = Packer()
            pk.add("n", n.astype(np.int32)).add("k", k.astype(np.int32))
            pk.add("noff", _off(n)).add("koff", _off(k))
            pk.add("dd_off", dd_off).add("ld_off", ld_off).add("lam_off", d.lam_off)
            for bi, sel in enumerate(_solve_buckets(n)):
                pk.add(f"sv{bi}", sel)
            t = pk.upload()
            levels.append(FactoredLevel(DevFactorLevel(n, k, dd_off, ld_off, d.lam_off, slabs[0],
                                                       slabs[1], slabs[2], d.Lam, d.child_off, t)))
        return FactoredInverse(levels, self.S_hat, self.S_inv, self.n, self.perm, self.scalar_field,
                               self.warnings)

    def factor_bytes(self):
        it = np.dtype(self.dtype).itemsize
        tot = 0
        for lv in self.levels:
            n, k = lv.dev.n, lv.dev.k
            tot += int((n * n + 2 * n * k).sum()) * it
        if self.S_inv is not None:
            tot += self.S_inv.numel() * it
        return tot


_BIG_TOP = 768          # top matrices above this size use the cooperative inverse


def factored_level_from_host(nodes, field):
    """Device level from host blocks [(Dd, Ld, Rd), ...] (a loaded container)."""
    torch = _native.require_cuda()
    dt = np.complex128 if field else np.float64
    n = np.array([Dd.shape[0] for Dd, _, _ in nodes], dtype=np.int64)
    k = np.array([Ld.shape[1] if Ld.ndim == 2 else 0 for _, Ld, _ in nodes], dtype=np.int64)
    dd_off, ld_off, lam_off = _off(n * n), _off(n * k), _off(np.zeros_like(k))
    cat = lambda arrs: (np.concatenate([np.asarray(a, dtype=dt).ravel() for a in arrs])  # noqa: E731
                        if arrs else np.zeros(0, dtype=dt))
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda")  # noqa: E731
    Dd = up(cat([x[0] for x in nodes]) if nodes else np.zeros(1, dt))
    Ld = up(cat([x[1] for x in nodes]) if nodes else np.zeros(1, dt))
    Rd = up(cat([x[2] for x in nodes]) if nodes else np.zeros(1, dt))
    Lam = torch.zeros(1, dtype=Dd.dtype, device="cuda")
    pk = Packer()
    pk.add("n", n.astype(np.int32)).add("k", k.astype(np.int32))
    pk.add("noff", _off(n)).add("koff", _off(k))
    pk.add("dd_off", dd_off).add("ld_off", ld_off).add("lam_off", lam_off)
    for bi, sel in enumerate(_solve_buckets(n)):
        pk.add(f"sv{bi}", sel)
    t = pk.upload()
    lv = FactoredLevel(DevFactorLevel(n, k, dd_off, ld_off, lam_off, Dd, Ld, Rd, Lam, None, t))
    lv._nodes = [FactoredNode(Dd=np.asarray(a, dtype=dt), Ld=np.asarray(b, dtype=dt),
                              Rd=np.asarray(c, dtype=dt), Lam=np.zeros((0, 0), dtype=dt))
                 for a, b, c in nodes]
    return lv


def _invert_top(Sh, regularize, field):
    """Shat^-1 on the device (single CTA Gauss-Jordan); status 1 -> singular."""
    torch = _native.require_cuda()
    K = Sh.shape[0]
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    if K > _BIG_TOP:
        # whole-GPU cooperative Gauss-Jordan (csrc/big.cu)
        L = _native.lib()
        scratch = torch.empty(int(L.skel_gj_scratch_bytes(K)) // 8 + 1, dtype=torch.float64,
                              device="cuda")
        _native.check(L.skel_dense_inverse_big(_native.ptr(Sh), K, float(regularize), _native.ptr(st),
                                               field, _native.ptr(scratch), _native.stream_ptr()),
                      "skel_dense_inverse_big")
        return int(st.item()), 1.0
    rc = torch.zeros(1, dtype=torch.float64, device="cuda")
    scratch = torch.empty((K * K + 3 * K) * (2 if field else 1) + 1, dtype=torch.float64, device="cuda")
    _native.check(_native.lib().skel_dense_inverse(_native.ptr(Sh), None, None, K, float(regularize),
                                                   _native.ptr(st), _native.ptr(rc), field,
                                                   _native.ptr(scratch), _native.stream_ptr()),
                  "skel_dense_inverse")
    return int(st.item()), float(rc.item())


class FactorRun:
    """Incremental telescoping factorization: ``add_level`` launches one
    level (size buckets on side streams) on ``stream`` without any host
    synchronisation; ``finish`` joins, maps the per-box statuses to the
    reference's exceptions / warnings and factors the top.  compress_source
    drives one of these on a side stream so level l's factor overlaps level
    l+1's compression."""

    def __init__(self, field, regularize=0.0, stream=None, shard=None):
        self.torch = _native.require_cuda()
        self.shard = shard
        self.field = field
        self.regularize = float(regularize)
        self.stream = stream
        self.levels = []       # (plan, DevFactorLevel, status, rcd, rcm, dl)
        self.keep = []

    def add_level(self, li, dl):
        torch = self.torch
        dev = torch.device("cuda")
        field = self.field
        tdt = _native.torch_dtype(field)
        elem = 16 if field else 8
        optin = _smem_optin()
        L = _native.lib()
        p_ = _native.ptr
        mine = getattr(dl, "mine", None)
        # sharded level: Dd / Ld / Rd slots for this rank's boxes only; the
        # Lambda slab keeps every box's slot (parents above the split read
        # it).  Offsets, classes, big boxes and launch buckets: csrc/plan.cpp
        pl = plan_factor_level(dl.nr, dl.nc, dl.kr, dl.kc, mine, elem, optin, _FAC_CLASSES,
                               _BIG_FAC_N, 400, _SOLVE_CLASSES)
        sq_bad, lam_bad, n, k = pl.sq_bad, pl.lam_bad, pl.n, pl.k
        n_own = n if mine is None else n * mine
        dd_off, ld_off, lam_off = pl.dd_off, pl.ld_off, pl.lam_off
        big = pl.big
        buckets = pl.buckets
        merged = pl.merged if pl.merged_first else None
        p = dl.p
        if self.stream is not None:
            # the compressed level's slabs and index arrays were allocated on the
            # caller's stream but are read by kernels queued on the eager stream:
            # tell the allocator, or dropping the compression without factor()
            # (nothing ever joins the eager stream then) lets the blocks be
            # reused while those kernels still run
            for x in (dl.D, dl.L, dl.R, *dl.t.values()):
                if hasattr(x, "record_stream") and x.is_cuda:
                    x.record_stream(self.stream)
        outer = torch.cuda.stream(self.stream) if self.stream is not None else _nullctx()
        with outer:
            pk = Packer()
            pk.add("n", n.astype(np.int32)).add("k", k.astype(np.int32))
            pk.add("noff", pl.noff).add("koff", pl.koff)
            pk.add("dd_off", dd_off).add("ld_off", ld_off).add("lam_off", lam_off)
            for bi, sel in enumerate(buckets):
                pk.add(f"order{bi}", sel)
            sv = pl.sbuckets
            for bi, sel in enumerate(sv):
                pk.add(f"sv{bi}", sel)
            t = pk.upload()
            Dd = torch.empty(max(int(dd_off[-1]), 1), dtype=tdt, device=dev)
            Ld = torch.empty(max(int(ld_off[-1]), 1), dtype=tdt, device=dev)
            Rd = torch.empty(max(int(ld_off[-1]), 1), dtype=tdt, device=dev)
            gather_lam = mine is not None and li == self.shard.split
            Lam = (torch.zeros if gather_lam else torch.empty)(max(int(lam_off[-1]), 1), dtype=tdt,
                                                               device=dev)
            status = torch.zeros(p, dtype=torch.int32, device=dev)
            rcd = torch.ones(p, dtype=torch.float64, device=dev)
            rcm = torch.ones(p, dtype=torch.float64, device=dev)
            fl = DevFactorLevel(n, k, dd_off, ld_off, lam_off, Dd, Ld, Rd, Lam, dl.child_off, t,
                                n_own=n_own, mine=mine, sv=sv)
            prev = self.levels[-1][1] if self.levels else None
            F = _native.SkelFactorLevel()
            F.nbox, F.level, F.regularize = p, li, self.regularize
            F.n, F.k = p_(fl.t_n), p_(fl.t_k)
            F.d_off, F.l_off, F.r_off = p_(dl.t_d_off), p_(dl.t_l_off), p_(dl.t_r_off)
            F.D, F.L, F.R = p_(dl.D), p_(dl.L), p_(dl.R)
            if li > 0:
                F.child_off = p_(dl.t_child_off)
                F.prev_lam_off, F.prev_lam, F.prev_k = p_(prev.t_lam_off), p_(prev.Lam), p_(prev.t_k)
            F.dd_off, F.ld_off, F.rd_off, F.lam_off = (p_(fl.t_dd_off), p_(fl.t_ld_off),
                                                       p_(fl.t_ld_off), p_(fl.t_lam_off))
            F.Dd, F.Ld, F.Rd, F.Lam = p_(Dd), p_(Ld), p_(Rd), p_(Lam)
            F.status, F.rcond_d, F.rcond_m = p_(status), p_(rcd), p_(rcm)
            streams = fork(len(buckets), tag="factor") if len(buckets) > 1 else None
            for bi, sel in enumerate(buckets):
                max_n = int(n[sel].max())
                max_k = int(k[sel].max())
                if merged is not None and bi == 0:
                    max_n, max_k = merged
                nd = (max_n * max_n + 4 * max_n * max_k + max_k * max_k + 4 * max_n + max_k) * elem   # fac_elems (factor.cu)
                F.order, F.nrun = p_(t[f"order{bi}"]), sel.size
                F.scratch, F.scratch_bytes = None, 0
                if nd + 1024 + 4 * max_n > optin:
                    scr = torch.empty(sel.size * nd // 8 + 1, dtype=torch.float64, device=dev)
                    self.keep.append(scr)
                    F.scratch, F.scratch_bytes = p_(scr), sel.size * nd
                rec = on_stream(streams[bi] if streams else torch.cuda.current_stream(),
                                lambda sp: _native.check(L.skel_factor_level(F, max_n, max_k, field, sp),
                                                         f"skel_factor_level ({li})"),
                                "factor_level", level=li)
                if rec is not None:
                    b_ = sel
                    nf, kf = n.astype(np.float64), k.astype(np.float64)
                    rec.flops = float((2 * nf[b_] ** 3 + 6 * nf[b_] ** 2 * kf[b_]
                                       + 6 * kf[b_] ** 2 * nf[b_] + 2 * kf[b_] ** 3).sum())
                    rec.nbytes = float(((nf[b_] ** 2 + 2 * nf[b_] * kf[b_]) * 2 + kf[b_] ** 2).sum()) * elem
            for a in np.nonzero(big)[0]:
                na, ka = int(n[a]), int(k[a])
                wb = int(L.skel_factor_big_bytes(na, ka, field))
                # allocated on this (the launching) stream: reuse is stream-ordered
                work = torch.empty(wb // 8 + 1, dtype=torch.float64, device=dev)
                with _profile.timed("factor_big", level=li):
                    _native.check(L.skel_factor_big(F, int(a), na, ka, int(dd_off[a]), int(ld_off[a]),
                                                    int(ld_off[a]), int(lam_off[a]), p_(work), wb, field,
                                                    _native.stream_ptr()), f"skel_factor_big ({li})")
            if streams:
                join(streams)
            if gather_lam:
                self.shard.gather_rows(Lam, lam_off, li)   # the split cover's Lambdas, everywhere
        self.levels.append(((sq_bad, lam_bad, n, k), fl, status, rcd, rcm, dl))

    def finish(self, cm):
        torch = self.torch
        if self.stream is not None:
            ev = torch.cuda.Event()
            ev.record(self.stream)
            torch.cuda.current_stream().wait_event(ev)
        warns = []
        flevels = []
        for li, (_, fl, status, rcd, rcm, _) in enumerate(self.levels):
            if fl.mine is not None:
                # the owned boxes' status / rcond estimates, everywhere
                self.shard.gather_boxes(status, li)
                self.shard.gather_boxes(rcd, li)
                self.shard.gather_boxes(rcm, li)
        # every level's status / rcond in one device->host copy
        if self.levels:
            cat_s = torch.cat([x[2] for x in self.levels]).cpu().numpy()
            cat_r = torch.cat([torch.cat([x[3], x[4]]) for x in self.levels]).cpu().numpy()
        so, ro = 0, 0
        for li, ((sq_bad, lam_bad, n, k), fl, status, rcd, rcm, dl) in enumerate(self.levels):
            p = status.numel()
            sts = cat_s[so:so + p]
            rd_h, rm_h = cat_r[ro:ro + p], cat_r[ro + p:ro + 2 * p]
            so, ro = so + p, ro + 2 * p
            fails = np.nonzero(sq_bad | lam_bad | (sts != 0))[0]
            if fails.size:
                a = int(fails[0])
                if sq_bad[a]:
                    raise InvalidInput(f"non-square D block ({dl.nr[a]}x{dl.nc[a]}) at level {li + 1}, "
                                       f"node {a}; compress with equalize_ranks=True")
                if sts[a] == 1:
                    raise SingularBlock(li + 1, a, "D")
                if lam_bad[a]:
                    raise InvalidInput(f"non-square Lambda block ({dl.kc[a]}x{dl.kr[a]}) at level "
                                       f"{li + 1}, node {a}; compress with equalize_ranks=True")
                raise SingularBlock(li + 1, a, "Lambda")
            for a in np.nonzero(((n > 0) & (rd_h < _RCOND_WARN)) | ((k > 0) & (rm_h < _RCOND_WARN)))[0]:
                if n[a] > 0 and rd_h[a] < _RCOND_WARN:
                    warns.append((li + 1, int(a), "D", float(rd_h[a])))
                if k[a] > 0 and rm_h[a] < _RCOND_WARN:
                    warns.append((li + 1, int(a), "Lambda", float(rm_h[a])))
            flevels.append(FactoredLevel(fl))
        prev = self.levels[-1][1]
        S = cm.device_S()
        if S.shape[0] != S.shape[1]:
            raise InvalidInput(f"non-square S block ({S.shape[0]}x{S.shape[1]}) at level top, node 0; "
                               "compress with equalize_ranks=True")
        # top: Shat = S with the last level's Lambdas on the diagonal blocks
        Sh = S.clone()
        kro = _off(prev.k)
        for a in range(prev.p):
            ka = int(prev.k[a])
            if ka:
                Sh[kro[a]:kro[a] + ka, kro[a]:kro[a] + ka] = \
                    prev.Lam[prev.lam_off[a]:prev.lam_off[a] + ka * ka].view(ka, ka)
        if Sh.numel() == 0:
            return FactoredInverse(flevels, Sh, None, cm.n, cm.perm.copy(), cm.scalar_field, warns,
                                   shard=self.shard)
        Sinv = Sh.clone()
        status, _ = _invert_top(Sinv, self.regularize, self.field)
        if status:
            raise SingularBlock("top", 0, "S")
        return FactoredInverse(flevels, Sh, Sinv, cm.n, _frozen(cm.perm), cm.scalar_field, warns,
                               shard=self.shard)


def factor(cm: CompressedMatrix, regularize: float = 0.0) -> FactoredInverse:
    """Telescoping inverse of a compressed matrix (solver.py:187-276).

    A CompressedMatrix produced by compress_source already carries an
    eager factorization launched level by level on a side stream (same
    kernels, regularize = 0); it is reused unless ``regularize`` differs or
    the host view of a level was materialised (and may have been edited)."""
    field = cm.field
    if cm.nlevels == 0:
        S = cm.device_S()
        warns = []
        if S.shape[0] != S.shape[1]:
            raise InvalidInput(f"non-square S block ({S.shape[0]}x{S.shape[1]}) at level top, "
                               "node 0; compress with equalize_ranks=True")
        if S.numel() == 0:
            return FactoredInverse([], None, None, cm.n, cm.perm.copy(), cm.scalar_field, warns)
        Sinv = S.clone()
        status, _ = _invert_top(Sinv, regularize, field)
        if status:
            raise SingularBlock("top", 0, "S")
        return FactoredInverse([], S, Sinv, cm.n, cm.perm.copy(), cm.scalar_field, warns)
    run = getattr(cm, "_eager", None)
    touched = any(lv._nodes is not None and lv.dev is not None and lv.dev_from_compress
                  for lv in cm.levels)
    if run is not None and float(regularize) == 0.0 and not touched and cm.S_dev is not None:
        cm._eager = None
        return run.finish(cm)
    if touched:
        for lv in cm.levels:
            if lv._nodes is not None:
                lv.dev = None          # re-pack from the (possibly edited) host view
    run = FactorRun(field, regularize, shard=getattr(cm, "shard", None))
    for li, dl in enumerate(cm.device_levels()):
        run.add_level(li, dl)
    return run.finish(cm)


def _smem_optin():
    from .skel import _smem_optin as f
    return f()


def solve(fi: FactoredInverse, b):
    """x = Dd1 b + Ld1 [ ... Shat^-1 ... ] Rd1 b for one or many RHS
    (solver.py:279-318).  numpy in -> numpy out; a CUDA tensor in -> CUDA
    tensor out (no host round trip)."""
    torch = _native.require_cuda()
    on_dev = hasattr(b, "is_cuda")
    ba = b if on_dev else np.asarray(b)
    if ba.shape[0] != fi.n:
        raise InvalidInput(f"length mismatch: system is {fi.n}, rhs {ba.shape[0]}")
    single = ba.ndim == 1
    bdt = (np.complex128 if ba.is_complex() else np.float64) if on_dev else ba.dtype
    dtype = np.result_type(fi.dtype, bdt)
    if dtype == np.complex128 and fi.dtype == np.float64:
        # real factorization, complex data: two real solves (linear)
        return solve(fi, ba.real) + 1j * solve(fi, ba.imag)
    field = int(dtype == np.complex128)
    if on_dev:
        B = ba.reshape(fi.n, -1).to(_native.torch_dtype(field)).contiguous()
    else:
        B = torch.from_numpy(np.ascontiguousarray(ba.reshape(fi.n, -1), dtype=dtype)).to("cuda")
    X = solve_device(fi, B, _private=not on_dev)
    if on_dev:
        return X[:, 0] if single else X
    x = _native.to_host(X)
    return x[:, 0] if single else x


def _sweep_launch(L, d, direction, u, v, out, Rn, field, urows=None, wrows=None):
    """One level of the up- or down-sweep: size buckets on side streams.
    urows / wrows: the finest level's fused gather / scatter (tree order)."""
    torch = _native.require_cuda()
    p_ = _native.ptr
    bks = d.solve_buckets
    if not bks:
        return
    streams = fork(len(bks), tag="solve") if len(bks) > 1 else None
    main = _native.stream_ptr()
    for bi, (order, cnt, mn, mk) in enumerate(bks):
        st = _native.c_vp(streams[bi].cuda_stream) if streams else main
        if direction == "up":
            if mk == 0:
                continue
            _native.check(L.skel_sweep_up_rows(cnt, p_(d.t_n), p_(d.t_k), p_(d.t_noff), p_(d.t_koff),
                                               p_(d.t_ld_off), p_(d.Rd), p_(u), p_(out), Rn, field,
                                               mn, mk, p_(order), p_(urows), st), "sweep_up")
        else:
            _native.check(L.skel_sweep_down_rows(cnt, p_(d.t_n), p_(d.t_k), p_(d.t_noff),
                                                 p_(d.t_koff), p_(d.t_dd_off), p_(d.Dd),
                                                 p_(d.t_ld_off), p_(d.Ld), p_(u), p_(v), p_(out), Rn,
                                                 field, mn, mk, p_(order), p_(urows), p_(wrows), st),
                          "sweep_down")
    if streams:
        join(streams)


def _sweep_work(rec, d, Rn, field, up):
    """Algorithmic flops / bytes of one sweep launch: factor
    blocks read once, vectors read and written once."""
    it = 16 if field else 8
    fl = 4 if field else 1
    n, k = d.n.astype(np.float64), d.k.astype(np.float64)
    if up:
        rec.flops = fl * 2.0 * Rn * float((n * k).sum())
        rec.nbytes = it * float((n * k).sum() + Rn * (n.sum() + k.sum()))
    else:
        rec.flops = fl * 2.0 * Rn * float((n * n + n * k).sum())
        rec.nbytes = it * float((n * n + n * k).sum() + Rn * (2 * n.sum() + k.sum()))


_GRAPH_CACHE = 4
_GRAPH_MAX_R = 64
# SKEL_SOLVE_GRAPH=0: never capture / replay (profiling: ncu times every
# sweep launch of an eager solve, but not kernel nodes of a replayed graph)
_NO_GRAPH = __import__("os").environ.get("SKEL_SOLVE_GRAPH", "1") == "0"


def _device_rhs(fi: FactoredInverse, B):
    """Validate / normalise a device RHS for the sweeps: (N, R) or (N,), on
    the GPU, the factorization's field (real B for a complex factorization is
    promoted), row-major contiguous.  Anything else is InvalidInput."""
    torch = _native.require_cuda()
    if not isinstance(B, torch.Tensor) or not B.is_cuda:
        raise InvalidInput("solve_device expects a CUDA tensor")
    if B.ndim not in (1, 2) or B.shape[0] != fi.n:
        raise InvalidInput(f"length mismatch: system is {fi.n}, rhs shape {tuple(B.shape)}")
    if B.dtype not in (torch.float64, torch.complex128, torch.float32, torch.complex64):
        raise InvalidInput(f"unsupported rhs dtype {B.dtype}")
    if B.ndim == 1:
        B = B.reshape(fi.n, 1)
    want = _native.torch_dtype(fi.field)
    if B.dtype != want:
        if B.is_complex() and fi.field == 0:
            raise InvalidInput("complex rhs with a real factorization: use solve() "
                               "(two real solves) or pass the real and imaginary parts")
        B = B.to(want)
    return B.contiguous()


def solve_device(fi: FactoredInverse, B, graph: bool = True, _private: bool = False):
    """Device-resident solve of an (N, R) CUDA tensor (original ordering).

    The ~30-40 launches of one solve (gather, per-level size-bucketed sweeps
    on side streams, top GEMM, scatter) are captured into a CUDA graph on the
    first repeat of a shape and replayed from then on.  When the SAME tensor
    object comes back (the multi-RHS reuse pattern) the graph is captured on
    that tensor itself and replays with no input copy (the cache holds a
    reference, so the storage cannot be recycled under the graph); other
    tensors of that shape -- and every call from ``solve()``, whose uploads
    are fresh temporaries (``_private``) -- are copied into a private-input
    graph.  A complex B with a real factorization runs as two real solves.
    The result is always a fresh tensor."""
    import weakref
    torch = _native.require_cuda()
    if (isinstance(B, torch.Tensor) and B.is_cuda and B.is_complex() and fi.field == 0
            and B.ndim in (1, 2) and B.shape[0] == fi.n):
        xr = solve_device(fi, B.real, graph, _private=True)
        xi = solve_device(fi, B.imag, graph, _private=True)
        return torch.complex(xr, xi)
    single = isinstance(B, torch.Tensor) and B.ndim == 1
    user = B
    B = _device_rhs(fi, B)
    if B is not user:
        _private = True                      # a converted copy: never bind a graph to it
    X = _solve_graph(fi, B, graph, _private, user, weakref)
    return X[:, 0] if single else X


def _solve_graph(fi, B, graph, private, user, weakref):
    torch = _native.require_cuda()
    if (not graph or _NO_GRAPH or _profile.enabled or torch.cuda.is_current_stream_capturing()
            or fi.shard is not None or B.shape[1] > _GRAPH_MAX_R):
        # many RHS: launch overhead is noise next to the sweeps, and the
        # graph's output copy would not be (8.6 GB at 2^20 x 1024)
        return _solve_device_eager(fi, B)
    key = (int(B.shape[1]), B.dtype)
    cache = fi.__dict__.setdefault("_graphs", {})
    seen = fi.__dict__.setdefault("_graph_seen", set())
    ent = None
    if not private:
        last = fi.__dict__.get("_last_user")
        fi.__dict__["_last_user"] = weakref.ref(user)
        ent = cache.get(("user", id(user)))
        if ent is not None and ent[1] is not user:
            ent = None                       # id() recycled by another object
        if ent is None and last is not None and last() is user:
            ent = cache[("user", id(user))] = _capture(fi, B, cache)   # same tensor again
    if ent is not None:
        g, _, static_X = ent
    else:
        ent = cache.get(key)
        if ent is None and key not in seen:
            # first solve with this shape runs eagerly; a repeat pays the
            # one-time capture and replays from then on
            seen.add(key)
            return _solve_device_eager(fi, B)
        if ent is None:
            static_B = torch.empty_like(B)
            static_B.copy_(B)
            ent = cache[key] = _capture(fi, static_B, cache)
        g, static_B, static_X = ent
        static_B.copy_(B)
    g.replay()
    return static_X.clone()


def _capture(fi, static_B, cache):
    torch = _native.require_cuda()
    _solve_device_eager(fi, static_B)          # warm-up: kernel attributes, allocator
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        static_X = _solve_device_eager(fi, static_B)
    while len(cache) >= _GRAPH_CACHE:
        cache.pop(next(iter(cache)))
    return g, static_B, static_X


def _solve_device_eager(fi: FactoredInverse, B):
    """Device-resident solve of an (N, R) CUDA tensor (original ordering)."""
    torch = _native.require_cuda()
    L = _native.lib()
    st = _native.stream_ptr()
    p_ = _native.ptr
    field = fi.field
    Rn = B.shape[1]
    perm = fi.perm_dev()
    # few RHS, one rank: the tree-order gather of B and scatter of X are fused
    # into the finest level's sweeps (row maps), no permuted copies
    fuse = bool(fi.levels) and fi.shard is None and Rn <= 16 and B.is_contiguous()
    if fuse:
        bt, rows = B, perm
    else:
        bt, rows = torch.empty_like(B), None
        _native.check(L.skel_permute_rows(p_(perm), fi.n, p_(B), p_(bt), Rn, 0, field, st), "permute")
    if not fi.levels:
        xt = _dense_apply(fi.S_inv, bt, field) if fi.S_inv is not None else bt
    else:
        us = [bt]
        u = bt
        shard = fi.shard
        for li, lv in enumerate(fi.levels):
            d = lv.dev
            sh = d.mine is not None
            nxt = torch.empty((int(d.k.sum()), Rn), dtype=B.dtype, device="cuda")
            with _profile.timed("sweep", dir="up") as rec:
                _sweep_launch(L, d, "up", u, None, nxt, Rn, field, urows=rows if li == 0 else None)
            if sh and li == shard.split:
                # split-level vector: every rank's rows, on every rank
                shard.gather_rows(nxt, _off(d.k), li)
            if rec is not None:
                _sweep_work(rec, d, Rn, field, up=True)
            us.append(nxt)
            u = nxt
        v = _dense_apply(fi.S_inv, u, field) if (fi.S_inv is not None and u.shape[0]) else u
        for li in range(len(fi.levels) - 1, -1, -1):
            d = fi.levels[li].dev
            sh = d.mine is not None
            last = li == 0 and fuse
            w = torch.empty((int(d.n.sum()), Rn), dtype=B.dtype, device="cuda")
            with _profile.timed("sweep", dir="down") as rec:
                _sweep_launch(L, d, "down", us[li], v, w, Rn, field, urows=rows if li == 0 else None,
                              wrows=rows if last else None)
            if sh and li == 0:
                shard.gather_rows(w, _off(d.n), 0)   # every rank's solution rows
            if rec is not None:
                _sweep_work(rec, d, Rn, field, up=False)
            v = w
        xt = v
        if fuse:
            return xt                                 # already in original order
    X = torch.empty_like(xt)
    _native.check(L.skel_permute_rows(p_(perm), fi.n, p_(xt), p_(X), Rn, 1, field, st), "permute")
    return X


# Names the reference defines in solver.py (sparse embedding + Matrix Market
# solver.py:91-140,414-433; GMRES 321-408; SKLC factorization files 439-529)
# live in embedding.py / krylov.py / container.py here; re-exported lazily
# (those modules import this one).
_ELSEWHERE = {
    "SparseEmbedding": "embedding", "assemble_embedding": "embedding",
    "export_matrix_market": "embedding", "read_matrix_market": "embedding",
    "gmres": "krylov",
    "serialize_factored": "container", "deserialize_factored": "container",
    "save_factored": "container", "load_factored": "container",
}


def __getattr__(name):
    mod = _ELSEWHERE.get(name)
    if mod is not None:
        import importlib
        return getattr(importlib.import_module(f"{__package__}.{mod}"), name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
