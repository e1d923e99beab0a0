"""Multi-rank (subtree-sharded) path, SURVEY.md 8(e).

CPU: two gloo ranks build the same ShardPlan (ownership contiguous per
level, children local, balanced) and exchange through its all-reduce.
GPU: two gloo ranks run the sharded compress / factor / solve / apply and
must reproduce the single-process results bit for bit (the per-box kernels
are the same; only which rank runs them changes).  Both ranks share the one
visible GPU; their kernels never wait on each other (the exchange is
host-side gloo)."""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "shard_worker.py")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(nproc, *args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), WORKER, *map(str, args)]
    env = dict(os.environ, OMP_NUM_THREADS="4")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_shard_plan_two_ranks(tmp_path):
    out = tmp_path / "plan.npz"
    _torchrun(2, "plan", out)
    d = np.load(out)
    assert int(d["split"]) > 0
    assert d["per"].min() > 0


def test_shard_plan_single_rank_owns_all():
    import paper_1110_3105_b200 as sk
    from paper_1110_3105_b200.shard import ShardPlan, default_plan
    t = np.linspace(0, 2 * np.pi, 8192, endpoint=False)
    tree = sk.build_tree(sk.PointSet(np.stack([2 * np.cos(t), np.sin(t)], 1)), 64)
    sp = ShardPlan(tree, 1, 0)
    for li in range(sp.split + 1):
        assert sp.mine(li).all()
    assert default_plan(tree) is None          # not a distributed job


@pytest.mark.gpu
@pytest.mark.parametrize("n,eps,world", [(16384, 1e-10, 2), (65536, 1e-12, 3)])
def test_sharded_solve_bit_identical(tmp_path, n, eps, world):
    import paper_1110_3105_b200 as sk
    from paper_1110_3105_b200 import bie
    out = tmp_path / "solve.npz"
    _torchrun(world, "solve", out, n, eps)
    d = np.load(out)
    curve = bie.ellipse(2.0, 1.0, n)
    system = bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
    tree, cm = bie.compress_system(system, eps, 64)
    fi = sk.factor(cm)
    B = np.random.default_rng(7).standard_normal((n, 3))
    X = sk.solve(fi, B)
    Y = sk.apply(cm, B[:, 0])
    kr = np.concatenate([lv.dev.kr for lv in cm.levels])
    assert int(d["split"]) >= 1
    np.testing.assert_array_equal(d["kr"], kr)
    np.testing.assert_array_equal(d["S"], cm.S_dev.cpu().numpy())
    np.testing.assert_array_equal(d["X"], X)
    np.testing.assert_array_equal(d["Xc"], X)
    np.testing.assert_array_equal(d["Y"], Y)
