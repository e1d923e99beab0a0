"""Multi-GPU sharding of the factor / solve path: subtree
sharding at a split level.

One process per GPU.  The boxes of a coarse "split" cover are cut into
`world` contiguous groups balanced by point count; every finer box belongs to
the rank that owns its ancestor in the split cover, so each rank's boxes form
one contiguous range per level and every box's children are local.  Per
level below (and at) the split, each rank compresses and factors only its own
boxes; the only exchanges are

  * after every sharded level: the per-box ranks / flags (p ints each) and
    the compacted skeleton lists -- neighbour boxes of a rank's boxes may
    live on another rank.  Each is an all_gather of the rank's OWNED
    contiguous range only (no zero-padded full-size reduction);
  * after the split level: the Lambda blocks of the split cover (the parents
    above it need them), an all_gather of the owned part of one small slab;
  * in the solve: the split-level vector after the up-sweep and the solution
    rows after the down-sweep.

Levels coarser than the split (a few hundred boxes at most) are computed
redundantly by every rank -- no gather / broadcast on the critical path.
The per-box kernels are identical to the single-GPU path, so results are
bit-identical for every world size.
"""

import numpy as np


class ShardPlan:
    def __init__(self, tree, world, rank, group=None, min_boxes_per_rank=16):
        self.world = int(world)
        self.rank = int(rank)
        self.group = group
        covers = tree.levels
        top = next(i for i, c in enumerate(covers) if len(c) == 1)
        # split: the coarsest cover (below the top) with enough boxes per rank
        split = 0
        for li in range(top):
            if covers[li].size >= min_boxes_per_rank * self.world:
                split = li
        self.split = split
        ids = covers[split]
        pts = (tree.hi[ids] - tree.lo[ids]).astype(np.float64)
        cum = np.cumsum(pts)
        # contiguous groups with ~equal point counts
        cuts = np.searchsorted(cum, cum[-1] * np.arange(1, self.world) / self.world, side="left")
        owner_split = np.zeros(ids.size, dtype=np.int64)
        for c in cuts:
            owner_split[c + 1:] += 1
        self.owner_split = owner_split
        split_lo = tree.lo[ids]
        self.owners = []
        for li in range(top):
            if li > split:
                self.owners.append(None)             # replicated level
                continue
            lo = tree.lo[covers[li]]
            anc = np.searchsorted(split_lo, lo, side="right") - 1
            self.owners.append(owner_split[anc])

    def box_range(self, li, q):
        """[b0, b1): the boxes rank q owns at sharded level li (contiguous)."""
        o = self.owners[li]
        return int(np.searchsorted(o, q, side="left")), int(np.searchsorted(o, q, side="right"))

    def bounds(self, off, li):
        """Per-rank [lo, hi) of an offset array over the level-li boxes."""
        out = []
        for q in range(self.world):
            b0, b1 = self.box_range(li, q)
            out.append((int(off[b0]), int(off[b1])))
        return out

    def all_gather_var(self, local, bounds, out):
        """out[bounds[q]] = rank q's ``local`` (rows; every rank's block is
        contiguous).  One all_gather of equal-size padded blocks."""
        import torch
        import torch.distributed as dist
        width = int(np.prod(out.shape[1:])) if out.dim() > 1 else 1
        flat = out.view(out.shape[0], width)
        mx = max(max(hi - lo for lo, hi in bounds), 1)
        lo, hi = bounds[self.rank]
        mine = torch.zeros((mx, width), dtype=out.dtype, device=out.device)
        mine[:hi - lo].copy_(local.reshape(hi - lo, width))
        if out.is_cuda and self._backend() == "gloo":
            parts = [torch.empty((mx, width), dtype=out.dtype) for _ in range(self.world)]
            dist.all_gather(parts, mine.cpu(), group=self.group)
            buf = torch.cat(parts).to(out.device)
        else:
            buf = torch.empty((self.world * mx, width), dtype=out.dtype, device=out.device)
            dist.all_gather_into_tensor(buf, mine, group=self.group)
        for q, (a, b) in enumerate(bounds):
            if b > a:
                flat[a:b].copy_(buf[q * mx:q * mx + (b - a)])
        return out

    def gather_rows(self, t, off, li):
        """All-gather of a row-sharded (rows, R) tensor: rank q holds rows
        off[b0_q]:off[b1_q] of the level-li box ranges; afterwards every rank
        holds all rows."""
        bd = self.bounds(off, li)
        lo, hi = bd[self.rank]
        return self.all_gather_var(t[lo:hi], bd, t)

    def gather_boxes(self, t, li, nseg=1):
        """``t`` holds ``nseg`` consecutive per-box segments over the level-li
        boxes (e.g. kr | kc | flags); every segment's owned box range is
        all-gathered into place with ONE collective."""
        import torch
        p = t.numel() // nseg
        v = t.view(nseg, p)
        bd = [self.box_range(li, q) for q in range(self.world)]
        b0, b1 = bd[self.rank]
        local = v[:, b0:b1].t().contiguous()
        full = torch.empty((p, nseg), dtype=t.dtype, device=t.device)
        self.all_gather_var(local, bd, full)
        v.copy_(full.t())
        return t

    def sharded(self, li):
        return li <= self.split

    def mine(self, li):
        """Boolean mask of this rank's boxes at level li (all True above the split)."""
        o = self.owners[li]
        if o is None:
            return None
        return o == self.rank

    # ---- collectives on device tensors -------------------------------------
    def _backend(self):
        import torch.distributed as dist
        return dist.get_backend(self.group)

    def all_reduce(self, t, op="sum"):
        """In-place all-reduce of a CUDA (or CPU) tensor over the plan's group
        (gloo: staged through host memory)."""
        import torch.distributed as dist
        rop = {"sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN,
               "max": dist.ReduceOp.MAX}[op]
        if t.is_cuda and self._backend() == "gloo":
            h = t.cpu()
            dist.all_reduce(h, op=rop, group=self.group)
            t.copy_(h.to(t.device))
        else:
            dist.all_reduce(t, op=rop, group=self.group)
        return t


def default_plan(tree):
    """ShardPlan for the current torch.distributed job, or None when not
    distributed / world size 1."""
    try:
        import torch.distributed as dist
    except Exception:
        return None
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return None
    return ShardPlan(tree, dist.get_world_size(), dist.get_rank())


__all__ = ["ShardPlan", "default_plan"]
