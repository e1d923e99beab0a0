#!/usr/bin/env python
"""Benchmark of the recursive-skeletonization factor / multi-RHS solve path
on B200 (BASELINE.json config 2 + config 5).

One step = one pass of the hot path over the config-2 workload: build the
quadtree + neighbour lists, compress (proxy IDs), factor (telescoping
inverse) of the 2D Laplace double-layer system on the a=2, b=1 ellipse at
N = 2^20, eps = 1e-12 (identity_coef -1/2), then a 16-RHS
solve.  ``value`` is the factor time (s) of the step (tree + compress +
factor, geometry resident in HBM), ``solve`` the 16-RHS N*RHS/s, and
``solve_1024`` config 5's 1024-RHS throughput on the same factorization.

  python bench.py [--gpus N --steps K --warmup W]      # ours
  python bench.py --impl reference ...                  # CPU oracle (rank 0)

Prints ONE JSON line on rank 0.  See DESIGN.md ("Measurement") for every key.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "factor time (s) and solve N·RHS/s at N=2^20, 1/2/4/8 GPU; rel err vs oracle"
CONFIG_NAME = ("config2: 2D Laplace double layer (identity_coef -1/2), ellipse a=2 b=1, "
               "N=2^20, eps=1e-12, leaf 64, 16 RHS; config5: same factor, 1024 RHS")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--points", dest="n", type=int, default=2 ** 20)
    ap.add_argument("--eps", type=float, default=1e-12)
    ap.add_argument("--nrhs", type=int, default=16)
    ap.add_argument("--nrhs-big", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-residual", action="store_true")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


SOLVES_PER_STEP = 10     # 16-RHS solves per timed solve step (mean reported)


def _ncu_traffic(name):
    """dram__bytes_read.sum + dram__bytes_write.sum of the committed
    `ncu --set full` capture of the dominant kernel (profiles/<name>, written
    by tools/profile_round.sh): bytes of that one launch."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", name)
    try:
        with open(path) as f:
            txt = f.read()
        head = txt.splitlines()[0].strip("- ")
        rd, wr = (float(x) for x in txt.split("dram bytes")[1].split()[:2])   # MB
        return (rd + wr) * 1e6, (f"profiles/{name}: one ncu --set full launch ({head[:60]}...), "
                                 f"DRAM read {rd:.1f} MB + write {wr:.1f} MB; FP64-bound kernel, "
                                 "targets are assembled in shared memory and never touch HBM")
    except Exception:
        return None, None


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.3)
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax = float(parts[2])
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU oracle (test infrastructure: the cpu_baseline leg / --impl reference)

def oracle_full(n, eps, nrhs, workers=None):
    """The reference algorithm on the host cores at the FULL workload size:
    oracle/ (numpy+scipy restatement of skelkit, pinned bit-exact to the live
    reference) with the boxes of each level farmed out to a process pool
    (oracle/parallel.py, the reference's _map_nodes structure).  Returns
    (factor seconds = tree + compress + factor, solve seconds for nrhs RHS,
    worker count, the factorization)."""
    import numpy as np

    import oracle
    from oracle.parallel import ParallelRun
    cur = oracle.ellipse(2.0, 1.0, n)
    t0 = time.perf_counter()
    T = oracle.build_tree(cur["xy"], 64)
    src = oracle.BieSource(cur, T.perm)
    with ParallelRun(src, T, eps, workers) as pr:
        of = pr.compress_factor()
        nw = pr.workers
    t1 = time.perf_counter()
    B = np.random.default_rng(0).standard_normal((n, nrhs))
    t2 = time.perf_counter()
    oracle.solve(of, B)
    t3 = time.perf_counter()
    return t1 - t0, t3 - t2, nw, of


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


REF_MAX_STEPS = 3        # full-size CPU steps take ~20 s each on 16 cores


def ref_description(nw):
    return (f"oracle/ (numpy+scipy restatement of skelkit 0.1.0, pinned bit-exact to the live "
            f"reference) at the FULL config-2 size, boxes of each level farmed to {nw} worker "
            f"processes (oracle/parallel.py = the reference's _map_nodes pool with processes, one "
            f"BLAS thread each); O(p) neighbour lists (the as-shipped O(p^2) scan would add "
            f"~5900 s at 2^20, SURVEY F4); compressed D/L/R stay in the workers")


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import warnings
    warnings.simplefilter("ignore")
    # warm-up: page in numpy/scipy and fork the pool once, on a small instance
    for _ in range(min(args.warmup, 1)):
        oracle_full(1 << 16, args.eps, args.nrhs)
    steps = max(1, min(args.steps, REF_MAX_STEPS))
    fts, sts = [], []
    nw = None
    for _ in range(steps):
        ft, stt, nw, _of = oracle_full(args.n, args.eps, args.nrhs)
        del _of
        fts.append(ft)
        sts.append(stt)
    ft = statistics.mean(fts)
    st = statistics.mean(sts)
    line = {
        "impl": "reference", "metric": METRIC, "value": ft, "unit": "s", "n_gpus": ws,
        "steps": steps, "warmup": min(args.warmup, 1), "steps_requested": args.steps,
        "warmup_requested": args.warmup, "ms_per_step": 1e3 * (ft + st),
        "value_steps": [round(t, 3) for t in fts],
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (analytic ellipse nodes, seeded N(0,1) RHS)",
        "config": config_dict(args),
        "solve": {"nrhs_per_s": args.n * args.nrhs / st, "R": args.nrhs, "ms": st * 1e3},
        "cpu_baseline": {"value": ft, "unit": "s", "cores": nw, "kind": "port",
                         "sample": ref_description(nw) + (
                             f"; {steps} full-size steps (capped at {REF_MAX_STEPS}), warm-up on "
                             f"N=2^16")},
        "e2e": {"value": ft, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(args):
    """Identical on both arms: the workload, not how it ran."""
    return {"workload": CONFIG_NAME, "n": args.n, "eps": args.eps, "nrhs": args.nrhs,
            "nrhs_big": args.nrhs_big,
            "l2": "GPU: 512 MB buffer written between timed steps; factor data 1.9 GB > L2"}


# ---------------------------------------------------------------------------
# ours

def fp64_peak(torch, lib, kind, iters=4096):
    import ctypes
    scratch = torch.zeros(4096, dtype=torch.float64, device="cuda")
    fl = ctypes.c_double()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    best = 0.0
    for _ in range(3):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        rc = lib.skel_fp64_probe(kind, iters, ctypes.c_void_p(scratch.data_ptr()), ctypes.byref(fl), st)
        e.record()
        torch.cuda.synchronize()
        if rc != 0:
            return None
        best = max(best, fl.value / (s.elapsed_time(e) * 1e-3) / 1e12)
    return best


def run_ours(args):
    import numpy as np
    import torch

    import paper_1110_3105_b200 as sk
    from paper_1110_3105_b200 import _native, _profile

    ws, rank, local = dist_env()
    torch.cuda.set_device(local % max(torch.cuda.device_count(), 1))
    dist = None
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = os.environ.get("SKEL_DIST_BACKEND", "nccl")   # gloo: code-path checks only
        if backend == "nccl":
            # communicator init lines (nRanks, NVLS / P2P transport) on stderr,
            # so the rank count of the NCCL job is checkable from the logs
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    import warnings
    warnings.simplefilter("ignore")
    n, eps, R = args.n, args.eps, args.nrhs
    curve = sk.bie.ellipse(2.0, 1.0, n)
    system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
    B_host = np.random.default_rng(0).standard_normal((n, R))
    # N>1: subtree-sharded factor (shard.py); every rank holds the whole RHS
    # block and solves its own boxes, the solution rows are all-gathered
    shard = "auto" if ws > 1 else None
    cols = np.arange(R)
    B_dev = torch.from_numpy(np.ascontiguousarray(B_host[:, cols])).to("cuda")
    flush = torch.empty(512 * 2 ** 20 // 8, dtype=torch.float64, device="cuda")   # > 126 MB L2

    def factor_step():
        tree = sk.build_tree(system.points, 64)
        src = sk.bie.BieSource(system, tree.perm)
        cm = sk.compress_source(src, tree, eps, shard=shard)
        return src, cm, sk.factor(cm)

    for _ in range(args.warmup):
        src, cm, fi = factor_step()
        sk.solve_device(fi, B_dev)
    torch.cuda.synchronize()

    clocks = ClockSampler(local % max(torch.cuda.device_count(), 1))
    clocks.start()
    fts, sts = [], []
    launches0 = _native.launch_count[0]
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        src, cm, fi = factor_step()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        fts.append(e0.elapsed_time(e1) * 1e-3)
    launches = _native.launch_count[0] - launches0
    # one extra factor step with per-launch CUDA events (outside the timed
    # steps: the events and per-launch stream switches cost host time)
    _profile.reset()
    _profile.enabled = True
    factor_step()
    torch.cuda.synchronize()
    _profile.enabled = False
    prof_steps = 1
    # the 16-RHS solve on the last factorization: the solve graph is captured
    # on the first repeat, then every timed solve is one graph replay
    # eager, capture, then warm replays: on a fresh box the first ~10 replays
    # after the factor steps run ~30 % slower (measured), so warm up a batch
    for _ in range(2 + max(3, args.warmup) * SOLVES_PER_STEP):
        sk.solve_device(fi, B_dev)
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        barrier()
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e1.record()
        for _ in range(SOLVES_PER_STEP):     # back to back: factor data (1.9 GB) >> L2
            X = sk.solve_device(fi, B_dev)
        e2.record()
        torch.cuda.synchronize()
        barrier()
        sts.append(e1.elapsed_time(e2) * 1e-3 / SOLVES_PER_STEP)
    clk = clocks.stop()
    factor_s = max_over_ranks(statistics.mean(fts))
    solve_s = max_over_ranks(statistics.mean(sts))
    # per-launch sweep events need the eager path (no graph): one extra solve
    _profile.enabled = True
    sk.solve_device(fi, B_dev, graph=False)
    torch.cuda.synchronize()
    _profile.enabled = False

    # roofline of the dominant kernel of the factor step, from the live events
    kinds = {}
    for kind in ("id_level", "factor_level", "sweep"):
        cnt, ms, flops, nbytes = _profile.summary(kind)
        kinds[kind] = (cnt, ms, flops, nbytes)
    kinds["id_level_union"] = _profile.union_ms("id_level", group="level")
    kinds["factor_level_union"] = _profile.union_ms("factor_level", group="level")
    pk_dfma = fp64_peak(torch, _native.lib(), 0)
    pk_dmma = fp64_peak(torch, _native.lib(), 1)
    fp64_pk = max(v for v in (pk_dfma, pk_dmma) if v)
    hbm_pk = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm_pk = float(json.load(f)["hbm_gbs"])
        hbm_src = "MEASURED_PEAKS.json"
    except Exception:
        hbm_pk, hbm_src = 6650.0, "fallback (B200_PROFILING.md)"
    cnt, ms, flops, _ = kinds["id_level"]
    ums = kinds["id_level_union"]
    # size buckets of one level run concurrently on side streams, so the
    # per-launch durations overlap: achieved = work / union of the launch
    # intervals per level (device time during which ID kernels were running)
    ach = flops / (ums * 1e-3) / 1e12 if ums > 0 else 0.0
    traffic, traffic_src = _ncu_traffic("r02/ncu_idbig.txt")
    roofline = {"kernel": "k_id_level (fused K1 assembly + K2 CPQR ID)", "bound": "fp64",
                "achieved": ach, "peak": fp64_pk, "unit": "TFLOP/s", "frac": ach / fp64_pk,
                "traffic": traffic, "traffic_source": traffic_src,
                "launches": cnt, "avg_launch_ms": ms / max(cnt, 1),
                "union_ms_per_step": ums / prof_steps,
                "share_of_factor": (ums * 1e-3 / prof_steps) / statistics.mean(fts),
                "peak_source": f"measured live by bench.py: DFMA {pk_dfma:.1f}, DMMA {pk_dmma:.1f} TFLOP/s "
                               "(MEASURED_PEAKS.json has no FP64 figure)",
                "work": "SURVEY 8(d): per box 2x[4mnk-2k^2(m+n)+k^2(n-k)] + 10 flop/entry assembly"}
    fc, fms, fflops, fbytes = kinds["factor_level"]
    sc, sms, sflops, sbytes = kinds["sweep"]
    # like the ID buckets, a level's factor buckets overlap on side streams:
    # achieved = work / union of the launch intervals per level
    fums = kinds["factor_level_union"]
    roof_factor = {"kernel": "k_factor_level", "bound": "fp64", "launches": fc,
                   "achieved": fflops / (fums * 1e-3) / 1e12 if fums else 0.0, "peak": fp64_pk,
                   "unit": "TFLOP/s", "union_ms_per_step": fums / prof_steps,
                   "launch_sum_ms_per_step": fms / prof_steps}
    roof_factor["frac"] = roof_factor["achieved"] / fp64_pk
    # algorithmic bytes of one solve, SURVEY 8(d) exactly: every factor block
    # read once (sum_a 8(n^2 + 2nk) + 8 K_top^2 = fi.factor_bytes()) plus B
    # read and X written once (16 N R), over the graph-replayed solve time.
    # The per-level vector round trips the sweeps actually make (each level
    # writes its u / w slab and the next reads it back) are reported beside
    # it as modelled traffic, not counted as useful bytes.
    alg_bytes = fi.factor_bytes() + 16.0 * n * len(cols)
    roof_solve = {"kernel": "k_level_dmma_few sweeps (R=%d), whole solve" % len(cols), "bound": "hbm",
                  "achieved": alg_bytes / solve_s / 1e9 if solve_s else 0.0, "peak": hbm_pk,
                  "unit": "GB/s", "peak_source": hbm_src, "launches": sc,
                  "bytes_per_solve": alg_bytes,
                  "bytes_rule": "SURVEY 8(d): factor blocks + 8 K_top^2 + 16 N R",
                  "traffic_model_bytes": sbytes,
                  "traffic_model_rule": "factor blocks + every level's vector slabs read/written",
                  "eager_launch_sum_gbs": sbytes / (sms * 1e-3) / 1e9 if sms else 0.0}
    roof_solve["frac"] = roof_solve["achieved"] / hbm_pk

    # config 5: 1024 RHS on the same factorization.  N>1: the sharded factor
    # is replicated once (one all-gather per slab, timed and reported), then
    # the RHS columns are sharded with no further traffic
    big = None
    if args.nrhs_big > 0:
        rep_ms = None
        fi_big = fi
        if ws > 1:
            torch.cuda.synchronize()
            barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            fi_big = fi.replicate()
            b.record()
            torch.cuda.synchronize()
            rep_ms = max_over_ranks(a.elapsed_time(b))
        bc = np.array_split(np.arange(args.nrhs_big), ws)[rank].size
        g = torch.Generator(device="cuda")
        g.manual_seed(1234 + rank)
        Bb = torch.randn((n, bc), dtype=torch.float64, device="cuda", generator=g)
        for _ in range(3):                 # warm-up (eager above 64 RHS: see solve_device)
            sk.solve_device(fi_big, Bb)
        torch.cuda.synchronize()
        ts = []
        for _ in range(max(2, min(args.steps, 4))):
            barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            sk.solve_device(fi_big, Bb)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        # per-launch sweep events (roofline) from one extra, eager solve
        _profile.reset()
        _profile.enabled = True
        sk.solve_device(fi_big, Bb, graph=False)
        torch.cuda.synchronize()
        _profile.enabled = False
        _, bms, bflops, bbytes = _profile.summary("sweep")
        tb = max_over_ranks(statistics.mean(ts))
        big = {"R": args.nrhs_big, "nrhs_per_s": n * args.nrhs_big / tb, "ms": tb * 1e3,
               "columns_per_rank": bc, "replicate_factor_ms": rep_ms,
               "roofline": {"kernel": "k_level_dmma_pipe sweeps, whole solve", "bound": "fp64",
                            "achieved": bflops / tb / 1e12 if tb else 0.0,
                            "peak": fp64_pk, "unit": "TFLOP/s", "flops_per_solve": bflops,
                            "eager_launch_sum_tfs": bflops / (bms * 1e-3) / 1e12 if bms else 0.0}}
        big["roofline"]["frac"] = big["roofline"]["achieved"] / fp64_pk
        del Bb, fi_big

    # end to end through the public API, host buffers in and out
    e2e_ts = []
    nrhs_local = len(cols)
    B_pinned = torch.from_numpy(np.ascontiguousarray(B_host[:, cols])).pin_memory().numpy()
    n_e2e = args.warmup + max(1, args.steps)
    for it in range(n_e2e):
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        sys_e = sk.bie.discretize_dirichlet(sk.bie.Curve2D(curve.t, curve.xy, curve.normals,
                                                           curve.curvature, curve.weights),
                                            sk.KernelSpec("laplace", 2))
        sigma, cm_e, fi_e = sk.bie.solve_dirichlet(sys_e, B_pinned, eps, 64, shard=shard)
        torch.cuda.synchronize()
        if it >= args.warmup:        # warm-up calls: pinned host pools, kernel attributes
            e2e_ts.append(time.perf_counter() - t0)
        del fi_e
        if it + 1 < n_e2e:
            del cm_e                 # the last call's compression feeds the parity report
    e2e_s = max_over_ranks(statistics.mean(e2e_ts))
    h2d = n * 8 * (2 + 2 + 1 + 1 + 1) + n * nrhs_local * 8
    d2h = n * nrhs_local * 8

    # correctness evidence at full size: residual against the exact operator
    resid = None
    if not args.no_residual and rank == 0:
        xs = np.asarray(sigma)[:, :1]
        y = sk.bie.dense_matvec(src, xs)
        bcol = B_host[:, cols[:1]]
        resid = float(np.linalg.norm(y - bcol) / np.linalg.norm(bcol))

    # SURVEY 8(d) correctness numbers against the live-reference fixture of
    # this exact config (tests/golden/make_golden_full.py): per-box rank
    # deltas, differing skeleton sets, solution error, both K6 residuals
    parity = None
    gpath = os.path.join(ROOT, "tests", "golden", "full_c2_ellipse_1048576_1e-12.npz")
    if (not args.no_residual and rank == 0 and ws == 1 and args.n == 1 << 20 and args.eps == 1e-12
            and os.path.exists(gpath)):
        sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
        from skelhash import skel_set_hash
        g = np.load(gpath)
        hist, diff_r, diff_c, worst = {}, 0, 0, 0
        for li in range(int(g["nlevels"])):
            lv = cm_e.levels[li]
            kr, kc = lv.kr_counts, lv.kc_counts
            dr = kr - g[f"L{li}_kr"].astype(np.int64)
            dc = kc - g[f"L{li}_kc"].astype(np.int64)
            for v, c_ in zip(*np.unique(np.concatenate([dr, dc]), return_counts=True)):
                hist[int(v)] = hist.get(int(v), 0) + int(c_)
            worst = max(worst, int(np.abs(dr).max(initial=0)), int(np.abs(dc).max(initial=0)))
            rs, cs = lv.skeleton_arrays()
            diff_r += int((skel_set_hash(rs, kr) != g[f"L{li}_row_hash"]).sum())
            diff_c += int((skel_set_hash(cs, kc) != g[f"L{li}_col_hash"]).sum())
        xr = g["X0"]
        x0 = np.asarray(sigma)[:, 0]
        yr = sk.bie.dense_matvec(src, xr.reshape(-1, 1))
        b0 = B_host[:, :1]
        parity = {"against": "live reference, tests/golden/full_c2_ellipse_1048576_1e-12.npz",
                  "rank_delta_hist": dict(sorted(hist.items())), "max_rank_delta": worst,
                  "row_skel_sets_differing": diff_r, "col_skel_sets_differing": diff_c,
                  "rel_err_x": float(np.linalg.norm(x0 - xr) / np.linalg.norm(xr)),
                  "residual_gpu": resid,
                  "residual_ref": float(np.linalg.norm(yr - b0) / np.linalg.norm(b0))}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        ft, st_, nw, _of = oracle_full(args.n, args.eps, R)
        del _of
        cpu = {"value": ft, "unit": "s", "cores": nw, "kind": "port",
               "sample": ref_description(nw) + "; one full-size step",
               "solve_nrhs_per_s": args.n * R / st_}

    if rank == 0:
        line = {
            "metric": METRIC, "value": factor_s, "unit": "s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * (factor_s + solve_s),
            "value_steps": [round(t, 5) for t in fts],
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (analytic ellipse nodes, seeded N(0,1) RHS)",
            "config": config_dict(args),
            "run": {"parallelism": ("single GPU" if ws == 1 else
                                    f"subtree-sharded factor over {ws} ranks below split level "
                                    f"{cm.shard.split}, replicated above; box-sharded solve"),
                    "levels": cm.nlevels, "S": list(cm.S_shape()),
                    "collectives": (None if dist is None else
                                    {"backend": dist.get_backend(), "world": dist.get_world_size(),
                                     "per_sharded_level": "all_gather(owned kr|kc|flags) + "
                                                          "all_gather(owned skeleton lists) x2"}),
                    "factor_bytes_per_point": fi.factor_bytes() / n},
            "solve": {"R": R, "nrhs_per_s": n * R / solve_s, "ms": solve_s * 1e3,
                      "solves_per_step": SOLVES_PER_STEP,
                      "ms_steps": [round(t * 1e3, 4) for t in sts]},
            "solve_1024": big,
            "roofline": roofline,
            "roofline_factor": roof_factor,
            "roofline_solve": roof_solve,
            "residual": resid,
            "parity": parity,
            "clocks": clk,
            "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "what": "bie.solve_dirichlet(host geometry, host 16-RHS) -> host solution"},
            "gpu_launches": launches,
            "gpu_launches_per_step": launches / max(args.steps, 1),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
