"""Worker for the multi-rank tests (launched by torch.distributed.run, one
process per rank, backend gloo).

  plan  <out>          CPU only: build the tree, the ShardPlan, check the
                       ownership invariants across ranks, the all-reduce and
                       the owned-range all-gathers.
  solve <out> <n> <eps> GPU: sharded compress -> factor -> solve / apply of
                       the 2D Laplace BIE (every rank on cuda:0 when only
                       one device is visible; the exchange is host-side
                       gloo, no kernel waits on another rank).
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _init():
    import torch.distributed as dist
    dist.init_process_group("gloo")
    return dist, dist.get_rank(), dist.get_world_size()


def plan(out):
    import torch
    import paper_1110_3105_b200 as sk
    from paper_1110_3105_b200.shard import ShardPlan
    dist, rank, world = _init()
    n = 1 << 16
    t = np.linspace(0, 2 * np.pi, n, endpoint=False)
    X = np.stack([2 * np.cos(t), np.sin(t)], 1)
    tree = sk.build_tree(sk.PointSet(X), 64)
    sp = ShardPlan(tree, world, rank)
    covers = tree.levels
    # same plan on every rank
    own_all = np.concatenate([o for o in sp.owners if o is not None]).astype(np.int64)
    g = [torch.zeros(own_all.size, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(g, torch.from_numpy(own_all))
    for x in g:
        assert np.array_equal(x.numpy(), own_all)
    for li in range(sp.split + 1):
        o = sp.owners[li]
        assert o.size == covers[li].size
        assert np.all(np.diff(o) >= 0), "ownership not contiguous"
        assert set(np.unique(o)) == set(range(world)), "a rank owns nothing"
        if li:
            ch = tree.cover_children(li)
            for a in range(o.size):
                assert np.all(sp.owners[li - 1][ch[a]:ch[a + 1]] == o[a]), "children not local"
    # load balance by points at the split cover
    ids = covers[sp.split]
    pts = tree.hi[ids] - tree.lo[ids]
    per = np.bincount(sp.owner_split, weights=pts, minlength=world)
    assert per.max() <= 1.5 * per.mean()
    t = torch.full((4,), float(rank + 1))
    sp.all_reduce(t)
    assert torch.all(t == world * (world + 1) / 2)
    m = torch.tensor([rank], dtype=torch.int32)
    sp.all_reduce(m, "max")
    assert int(m) == world - 1
    # row all-gather: rank q's rows of the level-0 point vector
    off = np.concatenate([[0], np.cumsum(tree.hi[covers[0]] - tree.lo[covers[0]])])
    v = torch.full((n, 2), -1.0)
    b0, b1 = sp.box_range(0, rank)
    v[off[b0]:off[b1]] = float(rank)
    sp.gather_rows(v, off, 0)
    want = np.repeat(sp.owners[0], np.diff(off)).astype(np.float64)
    assert np.array_equal(v[:, 0].numpy(), want) and np.array_equal(v[:, 1].numpy(), want)
    # per-box segments (kr | kc | flags layout): owned ranges gathered in place
    p1 = covers[1].size
    kk = torch.full((3 * p1,), -7, dtype=torch.int32)
    c0, c1 = sp.box_range(1, rank)
    for sgi in range(3):
        kk[sgi * p1 + c0:sgi * p1 + c1] = torch.arange(c0, c1, dtype=torch.int32) * 10 + sgi
    sp.gather_boxes(kk, 1, 3)
    want = (np.arange(p1)[None, :] * 10 + np.arange(3)[:, None]).reshape(-1)
    assert np.array_equal(kk.numpy(), want)
    if rank == 0:
        np.savez(out, split=sp.split, owners=own_all, per=per)
    dist.barrier()
    dist.destroy_process_group()


def solve(out, n, eps):
    import torch
    import paper_1110_3105_b200 as sk
    from paper_1110_3105_b200 import bie
    dist, rank, world = _init()
    torch.cuda.set_device(rank % torch.cuda.device_count())
    curve = bie.ellipse(2.0, 1.0, n)
    system = bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
    tree, cm = bie.compress_system(system, eps, 64, shard="auto")
    assert cm.shard is not None and cm.shard.world == world
    fi = sk.factor(cm)
    rng = np.random.default_rng(7)
    B = rng.standard_normal((n, 3))
    Xs = sk.solve(fi, B)
    Y = sk.apply(cm, B[:, 0])
    kr = np.concatenate([lv.dev.kr for lv in cm.levels])
    # replicated factor + column-sharded RHS (config-5 layout): rank r solves
    # columns r::world locally; gathered here only for the check
    fr = fi.replicate()
    assert fr.shard is None
    Xr = sk.solve(fr, B[:, rank::world])
    parts = [None] * world
    dist.all_gather_object(parts, Xr)
    Xc = np.empty_like(Xs)
    for q in range(world):
        Xc[:, q::world] = parts[q]
    if rank == 0:
        np.savez(out, X=Xs, Xc=Xc, Y=Y, kr=kr, split=cm.shard.split, S=cm.S_dev.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "plan":
        plan(sys.argv[2])
    else:
        solve(sys.argv[2], int(sys.argv[3]), float(sys.argv[4]))
