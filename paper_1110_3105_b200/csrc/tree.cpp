// tree.cpp -- native host builder of the adaptive orthtree, its covers and the
// same-cover neighbour lists (K7).
//
// Restates geom.py:118-184: root = padded bounding cube, centre splits with
// ties to the upper child, empty children pruned, subdivision stops at
// <= max_leaf points (or depth 60), DFS preorder node numbering and point
// permutation, covers with early leaves repeated at finer levels.
//
// Build: in-place stable counting sort of each node's point range into its
// 2^d children (coordinates are permuted alongside the indices so every pass
// streams), top levels serial, the subtrees below a frontier depth built in
// parallel on host threads and spliced back in preorder.
//
// Neighbours replace the reference's O(p^2) level_neighbors (geom.py:205-219)
// by a top-down O(p) search: two boxes of a cover can only touch if their
// cover-parents are equal or touch, so the candidates of a box are the
// children of its parent's neighbours; the reference predicate _boxes_touch
// (geom.py:187-189) then decides, and lists come out sorted -- identical to
// the reference's lists.
#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <condition_variable>
#include <functional>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/skel_b200.h"

namespace {

// Persistent worker pool: the tree build and the neighbour scan run several
// short parallel passes per call, and spawning 16 std::threads per pass cost
// more than some passes.  run(n, f) executes f(0..n-1) on the caller and the
// workers; nested calls (from a worker) run serially.  Every worker takes
// part in every generation, so no worker can touch a finished job.
class Pool {
 public:
  explicit Pool(int n) {
    for (int i = 0; i < n - 1; ++i) th_.emplace_back([this] { loop(); });
  }
  int size() const { return (int)th_.size() + 1; }
  void run(int n, const std::function<void(int)>& f) {
    if (in_worker() || th_.empty() || n <= 1) {
      for (int t = 0; t < n; ++t) f(t);
      return;
    }
    std::lock_guard<std::mutex> rl(run_m_);
    {
      std::lock_guard<std::mutex> l(m_);
      job_ = &f;
      njobs_ = n;
      next_ = 0;
      finished_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    in_worker() = true;          // a nested run() from the caller's share is serial
    for (int t; (t = next_.fetch_add(1)) < n;) f(t);
    in_worker() = false;
    std::unique_lock<std::mutex> l(m_);
    done_.wait(l, [&] { return finished_ == (int)th_.size(); });
  }

 private:
  static bool& in_worker() {
    thread_local bool w = false;
    return w;
  }
  void loop() {
    in_worker() = true;
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* j;
      int nj;
      {
        std::unique_lock<std::mutex> l(m_);
        cv_.wait(l, [&] { return gen_ != seen; });
        seen = gen_;
        j = job_;
        nj = njobs_;
      }
      for (int t; (t = next_.fetch_add(1)) < nj;) (*j)(t);
      std::lock_guard<std::mutex> l(m_);
      if (++finished_ == (int)th_.size()) done_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_, run_m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int njobs_ = 0, finished_ = 0;
  std::atomic<int> next_{0};
  uint64_t gen_ = 0;
};

// one pool per process, never destroyed (its threads die with the process)
static Pool& pool() {
  static Pool* p = [] {
    unsigned hwc = std::thread::hardware_concurrency();
    return new Pool((int)std::max(1u, std::min(hwc == 0 ? 1u : hwc, 32u)));
  }();
  return *p;
}


constexpr double kRootPad = 1e-12;
constexpr int kMaxDepth = 60;

struct NodeRec {
  double c[3];
  double hw;
  int64_t lo, hi, depth, parent;  // parent: local index within the owning list
  int64_t nchild;
};

struct Builder {
  int d;
  int64_t max_leaf;
  std::vector<int64_t>* perm;  // tree position -> original index
  double* px[3];               // coordinates in tree order (permuted alongside)
  std::vector<int64_t>* tmpi;
  std::vector<double>* tmpx[3];
  std::vector<uint8_t>* code;

  int nthreads = 1;

  // parallel stable counting sort of a large range (chunked per thread)
  void split_par(int64_t lo, int64_t hi, const double* cen, int64_t cnt[8]) {
    const int nk = 1 << d;
    const int T = nthreads;
    const int64_t len = hi - lo, chunk = (len + T - 1) / T;
    std::vector<std::array<int64_t, 8>> cc(T);
    uint8_t* cd = code->data();
    auto count = [&](int t) {
      std::array<int64_t, 8>& c = cc[t];
      c.fill(0);
      const int64_t a0 = lo + t * chunk, a1 = std::min(hi, a0 + chunk);
      for (int64_t i = a0; i < a1; ++i) {
        int k = 0;
        for (int a = 0; a < d; ++a) k |= (px[a][i] >= cen[a] ? 1 : 0) << a;
        cd[i] = (uint8_t)k;
        c[k]++;
      }
    };
    pool().run(T, count);
    std::vector<std::array<int64_t, 8>> st(T);
    int64_t s = lo;
    for (int k = 0; k < nk; ++k) {
      cnt[k] = 0;
      for (int t = 0; t < T; ++t) {
        st[t][k] = s;
        s += cc[t][k];
        cnt[k] += cc[t][k];
      }
    }
    int64_t* P = perm->data();
    int64_t* TI = tmpi->data();
    auto scatter = [&](int t) {
      std::array<int64_t, 8> pos = st[t];
      const int64_t a0 = lo + t * chunk, a1 = std::min(hi, a0 + chunk);
      for (int64_t i = a0; i < a1; ++i) {
        int64_t dst = pos[cd[i]]++;
        TI[dst] = P[i];
        for (int a = 0; a < d; ++a) (*tmpx[a])[dst] = px[a][i];
      }
    };
    pool().run(T, scatter);
    auto copyback = [&](int t) {
      const int64_t a0 = lo + t * chunk, a1 = std::min(hi, a0 + chunk);
      if (a1 <= a0) return;
      std::memcpy(P + a0, TI + a0, (a1 - a0) * sizeof(int64_t));
      for (int a = 0; a < d; ++a) std::memcpy(px[a] + a0, tmpx[a]->data() + a0, (a1 - a0) * sizeof(double));
    };
    pool().run(T, copyback);
  }

  // split [lo, hi) of node `cen/hw` into children ranges; returns counts
  void split(int64_t lo, int64_t hi, const double* cen, int64_t cnt[8]) {
    if (nthreads > 1 && hi - lo >= (int64_t)1 << 17) {
      split_par(lo, hi, cen, cnt);
      return;
    }
    const int nk = 1 << d;
    for (int c = 0; c < nk; ++c) cnt[c] = 0;
    uint8_t* cd = code->data();
    for (int64_t t = lo; t < hi; ++t) {
      int k = 0;
      for (int a = 0; a < d; ++a) k |= (px[a][t] >= cen[a] ? 1 : 0) << a;
      cd[t] = (uint8_t)k;
      cnt[k]++;
    }
    int64_t start[8];
    int64_t s = lo;
    for (int c = 0; c < nk; ++c) { start[c] = s; s += cnt[c]; }
    int64_t* P = perm->data();
    int64_t* TI = tmpi->data();
    for (int64_t t = lo; t < hi; ++t) {
      int64_t dst = start[cd[t]]++;
      TI[dst] = P[t];
      for (int a = 0; a < d; ++a) (*tmpx[a])[dst] = px[a][t];
    }
    std::memcpy(P + lo, TI + lo, (hi - lo) * sizeof(int64_t));
    for (int a = 0; a < d; ++a) std::memcpy(px[a] + lo, tmpx[a]->data() + lo, (hi - lo) * sizeof(double));
  }

  // serial preorder build of a subtree into `out` (parent indices local)
  void build_sub(std::vector<NodeRec>& out, int64_t lo, int64_t hi, const double* cen, double hw,
                 int64_t depth, int64_t parent) {
    const int64_t me = (int64_t)out.size();
    NodeRec r;
    for (int a = 0; a < 3; ++a) r.c[a] = a < d ? cen[a] : 0.0;
    r.hw = hw; r.lo = lo; r.hi = hi; r.depth = depth; r.parent = parent; r.nchild = 0;
    out.push_back(r);
    if (hi - lo <= max_leaf || depth >= kMaxDepth) return;
    int64_t cnt[8];
    split(lo, hi, cen, cnt);
    int64_t s = lo;
    for (int c = 0; c < (1 << d); ++c) {
      if (cnt[c] == 0) continue;
      double cc[3];
      for (int a = 0; a < d; ++a) cc[a] = cen[a] + (((c >> a) & 1) ? 0.5 : -0.5) * hw;
      out[me].nchild += 1;
      build_sub(out, s, s + cnt[c], cc, 0.5 * hw, depth + 1, me);
      s += cnt[c];
    }
  }
};

struct Tree {
  int dim = 2;
  int64_t n = 0;
  std::vector<double> center;  // nnodes * dim
  std::vector<double> hw;
  std::vector<int64_t> lo, hi, depth, parent, nchild;
  std::vector<int64_t> perm;
  std::vector<std::vector<int64_t>> covers;             // finest first
  std::vector<std::vector<int64_t>> nbr_off, nbr_idx;   // per cover
  bool nbr_done = false;
  std::thread nbr_thread;      // neighbour lists computed in the background after build
  std::mutex nbr_m;            // serialises the join of nbr_thread
  bool nonfinite = false;      // build() saw a NaN / inf coordinate
};

// Item of the serial top part: a node, or a subtree task spliced in later.
struct TopItem {
  bool task;
  NodeRec rec;        // node record (task: root geometry)
  int64_t parent_item;
};

static double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

void build(Tree& T, const double* X, int64_t n, int d, int64_t max_leaf) {
  const bool timing = getenv("SKEL_TREE_TIMING") != nullptr;
  double t0 = now_ms();
  T.dim = d;
  T.n = n;
  unsigned hwc = std::thread::hardware_concurrency();
  const int nthreads = (int)std::max(1u, std::min(hwc == 0 ? 1u : hwc, 32u));
  auto parallel = [&](auto fn) {        // fn(t, a0, a1) over point chunks
    const int64_t chunk = (n + nthreads - 1) / nthreads;
    pool().run(nthreads, [&](int t) {
      fn(t, std::min(n, (int64_t)t * chunk), std::min(n, (int64_t)(t + 1) * chunk));
    });
  };
  // bounding box (per-thread extrema, then reduced)
  // (and the finiteness check of geom.py:133, in the same pass)
  std::vector<std::array<double, 6>> ext_t(nthreads);
  std::vector<char> bad_t(nthreads, 0);
  parallel([&](int t, int64_t a0, int64_t a1) {
    std::array<double, 6> e = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    bool bad = false;
    for (int64_t i = a0; i < a1; ++i)
      for (int a = 0; a < d; ++a) {
        const double v = X[i * d + a];
        bad |= !std::isfinite(v);
        e[a] = std::min(e[a], v);
        e[3 + a] = std::max(e[3 + a], v);
      }
    ext_t[t] = e;
    bad_t[t] = bad;
  });
  for (int t = 0; t < nthreads; ++t)
    if (bad_t[t]) {
      T.nonfinite = true;
      return;
    }
  double lo_c[3] = {INFINITY, INFINITY, INFINITY}, hi_c[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int t = 0; t < nthreads; ++t)
    for (int a = 0; a < d; ++a) {
      lo_c[a] = std::min(lo_c[a], ext_t[t][a]);
      hi_c[a] = std::max(hi_c[a], ext_t[t][3 + a]);
    }
  double c0[3] = {0, 0, 0}, ext = 0.0, cabs = 0.0;
  for (int a = 0; a < d; ++a) {
    c0[a] = 0.5 * (lo_c[a] + hi_c[a]);
    ext = std::max(ext, hi_c[a] - lo_c[a]);
    cabs = std::max(cabs, std::fabs(c0[a]));
  }
  double hw0 = 0.5 * ext;
  double scale = std::max(std::max(hw0, cabs), 1.0);
  hw0 = hw0 * (1.0 + kRootPad) + kRootPad * scale;

  // scratch buffers are cached across builds: fresh multi-MB allocations
  // cost more in first-touch page faults than the whole partitioning
  static std::mutex scratch_mu;
  static std::vector<int64_t> s_tmpi;
  static std::vector<double> s_px[3], s_tmpx[3];
  static std::vector<uint8_t> s_code;
  static std::vector<uint16_t> s_top;
  std::lock_guard<std::mutex> guard(scratch_mu);
  std::vector<int64_t> perm(n);
  std::vector<int64_t>& tmpi = s_tmpi;
  if ((int64_t)tmpi.size() < n) tmpi.resize(n);
  std::vector<double>* pxv = s_px;
  std::vector<double>* tmpx = s_tmpx;
  for (int a = 0; a < d; ++a) {
    if ((int64_t)pxv[a].size() < n) pxv[a].resize(n);
    if ((int64_t)tmpx[a].size() < n) tmpx[a].resize(n);
  }
  std::vector<uint8_t>& code = s_code;
  if ((int64_t)code.size() < n) code.resize(n);
  Builder B;
  B.d = d;
  B.max_leaf = max_leaf;
  B.perm = &perm;
  B.tmpi = &tmpi;
  B.code = &code;
  for (int a = 0; a < 3; ++a) {
    B.px[a] = a < d ? pxv[a].data() : nullptr;
    B.tmpx[a] = &tmpx[a];
  }
  B.nthreads = nthreads;
  const int64_t frontier_size = std::max<int64_t>(4 * max_leaf, n / (4 * nthreads));

  double t0b = now_ms();
  // ---- top part, all at once: every point's child digits for the first DT
  // levels (the same centre arithmetic as the node splits, so the same
  // comparisons), one histogram, per-level counts, the depth at which each
  // top cell stops (leaf, or subtree task), and ONE stable counting sort by
  // the stopping prefix -- points of a node end up in original order, the
  // nodes in preorder, exactly as the recursive stable partitioning leaves them.
  const int DT = d == 2 ? 6 : 4;
  const int NB = 1 << (d * DT);
  std::vector<uint16_t>& tcode = s_top;
  if ((int64_t)tcode.size() < n) tcode.resize(n);
  std::vector<std::vector<int64_t>> hist_t(nthreads, std::vector<int64_t>(NB, 0));
  parallel([&](int t, int64_t a0, int64_t a1) {
    std::vector<int64_t>& h = hist_t[t];
    for (int64_t i = a0; i < a1; ++i) {
      double cen[3] = {c0[0], c0[1], c0[2]};
      double hw = hw0;
      unsigned cd = 0;
      for (int lev = 0; lev < DT; ++lev) {
        unsigned k = 0;
        for (int a = 0; a < d; ++a) k |= (X[i * d + a] >= cen[a] ? 1u : 0u) << a;
        cd = (cd << d) | k;
        for (int a = 0; a < d; ++a) cen[a] = cen[a] + (((k >> a) & 1) ? 0.5 : -0.5) * hw;
        hw = 0.5 * hw;
      }
      tcode[i] = (uint16_t)cd;
      h[cd]++;
    }
  });
  // counts of every prefix at every depth 0..DT
  std::vector<std::vector<int64_t>> cnt(DT + 1);
  cnt[DT].assign(NB, 0);
  for (int t = 0; t < nthreads; ++t)
    for (int b = 0; b < NB; ++b) cnt[DT][b] += hist_t[t][b];
  for (int l = DT - 1; l >= 0; --l) {
    cnt[l].assign((size_t)1 << (d * l), 0);
    for (size_t q = 0; q < cnt[l + 1].size(); ++q) cnt[l][q >> d] += cnt[l + 1][q];
  }
  auto stops = [&](int l, int64_t c) {
    const bool leaf = c <= max_leaf || l >= kMaxDepth;
    return leaf || c <= frontier_size || l == DT;
  };
  // sort key of each top cell: its stopping prefix, left-aligned
  std::vector<int32_t> key(NB);
  for (int b = 0; b < NB; ++b) {
    int l = 0;
    while (!stops(l, cnt[l][b >> (d * (DT - l))])) ++l;
    const int sh = d * (DT - l);
    key[b] = (b >> sh) << sh;
  }
  // stable counting sort by key: per-thread counts, key-major offsets
  std::vector<std::vector<int64_t>> kc_t(nthreads, std::vector<int64_t>(NB, 0));
  parallel([&](int t, int64_t a0, int64_t a1) {
    std::vector<int64_t>& c = kc_t[t];
    for (int64_t i = a0; i < a1; ++i) c[key[tcode[i]]]++;
  });
  {
    int64_t run = 0;
    for (int b = 0; b < NB; ++b)
      for (int t = 0; t < nthreads; ++t) {
        const int64_t c = kc_t[t][b];
        kc_t[t][b] = run;
        run += c;
      }
  }
  parallel([&](int t, int64_t a0, int64_t a1) {
    std::vector<int64_t>& pos = kc_t[t];
    for (int64_t i = a0; i < a1; ++i) {
      const int64_t dst = pos[key[tcode[i]]]++;
      perm[dst] = i;
      for (int a = 0; a < d; ++a) pxv[a][dst] = X[i * d + a];
    }
  });
  // the top nodes, in preorder over the prefix counts
  struct TNode {
    NodeRec rec;
    bool task, leaf;
    std::vector<int64_t> kids;
  };
  std::vector<TNode> top;
  {
    struct Frame { int l; int64_t q, lo, parent; double c[3]; double hw; };
    std::vector<Frame> st;
    Frame f0{0, 0, 0, -1, {c0[0], c0[1], c0[2]}, hw0};
    st.push_back(f0);
    while (!st.empty()) {
      Frame f = st.back();
      st.pop_back();
      const int64_t c = cnt[f.l][f.q];
      TNode t;
      for (int a = 0; a < 3; ++a) t.rec.c[a] = a < d ? f.c[a] : 0.0;
      t.rec.hw = f.hw; t.rec.lo = f.lo; t.rec.hi = f.lo + c; t.rec.depth = f.l;
      t.rec.parent = f.parent; t.rec.nchild = 0;
      t.leaf = c <= max_leaf || f.l >= kMaxDepth;
      t.task = !t.leaf && stops(f.l, c);
      const int64_t id = (int64_t)top.size();
      top.push_back(t);
      if (f.parent >= 0) {
        top[f.parent].kids.push_back(id);
        top[f.parent].rec.nchild += 1;
      }
      if (t.leaf || t.task) continue;
      // children pushed in reverse so they are visited (and numbered) in code order
      int64_t offs[8];
      int64_t off = f.lo;
      const int nk = 1 << d;
      for (int k = 0; k < nk; ++k) { offs[k] = off; off += cnt[f.l + 1][(f.q << d) | k]; }
      for (int k = nk - 1; k >= 0; --k) {
        const int64_t cc = cnt[f.l + 1][(f.q << d) | k];
        if (cc == 0) continue;
        Frame g;
        g.l = f.l + 1; g.q = (f.q << d) | k; g.lo = offs[k]; g.parent = id;
        for (int a = 0; a < 3; ++a) g.c[a] = a < d ? f.c[a] + (((k >> a) & 1) ? 0.5 : -0.5) * f.hw : 0.0;
        g.hw = 0.5 * f.hw;
        st.push_back(g);
      }
    }
  }
  // preorder item list of the top part (children in code order)
  std::vector<TopItem> items;
  {
    std::vector<std::pair<int64_t, int64_t>> st = {{0, -1}};   // (top node, parent item)
    while (!st.empty()) {
      auto [id, pitem] = st.back();
      st.pop_back();
      TopItem it;
      it.rec = top[id].rec;
      it.task = top[id].task;
      it.parent_item = pitem;
      const int64_t me = (int64_t)items.size();
      items.push_back(it);
      const std::vector<int64_t>& ks = top[id].kids;
      for (auto r = ks.rbegin(); r != ks.rend(); ++r) st.push_back({*r, me});
    }
  }
  double t1 = now_ms();
  // parallel subtrees (ranges are disjoint, so the in-place sorts do not race)
  std::vector<int64_t> task_ids;
  for (int64_t i = 0; i < (int64_t)items.size(); ++i)
    if (items[i].task) task_ids.push_back(i);
  std::vector<std::vector<NodeRec>> sub(task_ids.size());
  {
    pool().run((int)task_ids.size(), [&](int t) {
      const NodeRec& r = items[task_ids[t]].rec;
      B.build_sub(sub[t], r.lo, r.hi, r.c, r.hw, r.depth, -1);
    });
  }
  double t2 = now_ms();
  // splice in preorder
  std::vector<int64_t> item_gid(items.size());
  int64_t gid = 0;
  size_t tk = 0;
  for (size_t i = 0; i < items.size(); ++i) {
    item_gid[i] = gid;
    gid += items[i].task ? (int64_t)sub[tk++].size() : 1;
  }
  const int64_t nn = gid;
  T.center.resize(nn * d);
  T.hw.resize(nn);
  T.lo.resize(nn);
  T.hi.resize(nn);
  T.depth.resize(nn);
  T.parent.resize(nn);
  T.nchild.resize(nn);
  auto put = [&](int64_t g, const NodeRec& r, int64_t par) {
    for (int a = 0; a < d; ++a) T.center[g * d + a] = r.c[a];
    T.hw[g] = r.hw; T.lo[g] = r.lo; T.hi[g] = r.hi; T.depth[g] = r.depth;
    T.parent[g] = par; T.nchild[g] = r.nchild;
  };
  tk = 0;
  for (size_t i = 0; i < items.size(); ++i) {
    const int64_t par = items[i].parent_item >= 0 ? item_gid[items[i].parent_item] : -1;
    if (!items[i].task) {
      put(item_gid[i], items[i].rec, par);
    } else {
      const std::vector<NodeRec>& s = sub[tk++];
      const int64_t base = item_gid[i];
      for (size_t j = 0; j < s.size(); ++j)
        put(base + (int64_t)j, s[j], j == 0 ? par : base + s[j].parent);
    }
  }
  T.perm = std::move(perm);
  double t3 = now_ms();
  // covers in id order == sorted by range start (preorder, disjoint ranges)
  int64_t maxd = 0;
  for (int64_t i = 0; i < nn; ++i) maxd = std::max(maxd, T.depth[i]);
  T.covers.assign(maxd + 1, {});
  // node i lies in cover f iff depth == f, or it is a leaf shallower than f;
  // visiting nodes in id order keeps every cover sorted by range start
  for (int64_t i = 0; i < nn; ++i) {
    const int64_t f1 = T.nchild[i] == 0 ? maxd : T.depth[i];
    for (int64_t f = T.depth[i]; f <= f1; ++f) T.covers[maxd - f].push_back(i);
  }
  if (timing)
    fprintf(stderr, "tree: setup %.2f ms, top %.2f, subtrees %.2f ms (%zu tasks, %d threads), splice %.2f ms, covers %.2f ms\n",
            t0b - t0, t1 - t0b, t2 - t1, task_ids.size(), nthreads, t3 - t2, now_ms() - t3);
}

inline bool touch(const Tree& T, int64_t na, int64_t nb, double tol) {
  const int d = T.dim;
  for (int a = 0; a < d; ++a) {
    double gap = std::fabs(T.center[na * d + a] - T.center[nb * d + a]) - (T.hw[na] + T.hw[nb]);
    if (!(gap <= tol)) return false;
  }
  return true;
}

void all_neighbors(Tree& T) {
  if (T.nbr_done) return;
  const bool timing = getenv("SKEL_TREE_TIMING") != nullptr;
  const double tn0 = now_ms();
  const int nc = (int)T.covers.size();
  T.nbr_off.assign(nc, {});
  T.nbr_idx.assign(nc, {});
  const double tol = 1e-9 * T.hw[0];
  // top cover(s) with a single node: no neighbours
  for (int li = nc - 1; li >= 0; --li) {
    const std::vector<int64_t>& ids = T.covers[li];
    const int64_t p = (int64_t)ids.size();
    std::vector<int64_t>& off = T.nbr_off[li];
    std::vector<int64_t>& idx = T.nbr_idx[li];
    off.assign(p + 1, 0);
    idx.clear();
    if (li == nc - 1 || p < 2) continue;
    // cover parent of every node: the node of cover li+1 containing it
    const std::vector<int64_t>& up = T.covers[li + 1];
    const int64_t q = (int64_t)up.size();
    std::vector<int64_t> cstart(q + 1);  // children runs of cover li+1 in cover li
    int64_t j = 0;
    for (int64_t u = 0; u < q; ++u) {
      cstart[u] = j;
      while (j < p && T.lo[ids[j]] < T.hi[up[u]]) ++j;
    }
    cstart[q] = p;
    std::vector<int64_t> par(p);
    for (int64_t u = 0; u < q; ++u)
      for (int64_t t = cstart[u]; t < cstart[u + 1]; ++t) par[t] = u;
    const std::vector<int64_t>& uoff = T.nbr_off[li + 1];
    const std::vector<int64_t>& uidx = T.nbr_idx[li + 1];
    // candidates of boxes a0..a1: the children of the cover parent and of
    // the parent's neighbours, sorted; appended to out, counts per box
    auto scan = [&](int64_t a0, int64_t a1, std::vector<int64_t>& out, int64_t* cnt) {
      std::vector<int64_t> cand;
      for (int64_t a = a0; a < a1; ++a) {
        cand.clear();
        const int64_t u = par[a];
        auto take = [&](int64_t w) {
          for (int64_t t = cstart[w]; t < cstart[w + 1]; ++t)
            if (t != a && touch(T, ids[a], ids[t], tol)) cand.push_back(t);
        };
        take(u);
        for (int64_t s = uoff[u]; s < uoff[u + 1]; ++s) take(uidx[s]);
        std::sort(cand.begin(), cand.end());
        out.insert(out.end(), cand.begin(), cand.end());
        cnt[a - a0] = (int64_t)cand.size();
      }
    };
    std::vector<int64_t> cnt(p);
    unsigned hwc = std::thread::hardware_concurrency();
    const int nt = p >= 4096 ? (int)std::max(1u, std::min(hwc == 0 ? 1u : hwc, 16u)) : 1;
    if (nt == 1) {
      scan(0, p, idx, cnt.data());
    } else {
      // boxes are independent given the parent cover's lists: chunks in
      // parallel, concatenated in box order (identical to the serial lists)
      const int64_t chunk = (p + nt - 1) / nt;
      std::vector<std::vector<int64_t>> part(nt);
      pool().run(nt, [&](int t) {
        const int64_t a0 = std::min(p, t * chunk), a1 = std::min(p, (t + 1) * chunk);
        scan(a0, a1, part[t], cnt.data() + a0);
      });
      size_t tot = 0;
      for (auto& v : part) tot += v.size();
      idx.reserve(tot);
      for (auto& v : part) idx.insert(idx.end(), v.begin(), v.end());
    }
    for (int64_t a = 0; a < p; ++a) off[a + 1] = off[a] + cnt[a];
    if (timing) fprintf(stderr, "nbr level %d: %lld boxes, %d threads, %.2f ms since start\n", li,
                        (long long)p, nt, now_ms() - tn0);
  }
  T.nbr_done = true;
}


// numpy's pairwise summation of float64 (the add.reduce inner loop of a
// contiguous array: < 8 elements sequentially, <= 128 with 8 accumulators
// combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus the tail, otherwise
// split at n/2 rounded down to a multiple of 8), over w[perm[0..n)]
static double pw_sum(const double* w, const int64_t* perm, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += w[perm[i]];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = w[perm[j]];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += w[perm[i + j]];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += w[perm[i]];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pw_sum(w, perm, n2) + pw_sum(w + 0, perm + n2, n - n2);
}

// the same sum with the top recursion levels' subtrees summed on the pool:
// leaves (in order) are ranges the recursion reaches at `depth` or at
// <= 8192 elements; combining them back along the same splits keeps
// numpy's association exactly
static void pw_leaves(int64_t a, int64_t n, int depth, std::vector<std::pair<int64_t, int64_t>>& out) {
  if (depth == 0 || n <= 8192) {
    out.push_back({a, n});
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  pw_leaves(a, n2, depth - 1, out);
  pw_leaves(a + n2, n - n2, depth - 1, out);
}
static double pw_combine(int64_t n, int depth, const double* sums, size_t& k) {
  if (depth == 0 || n <= 8192) return sums[k++];
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  const double x = pw_combine(n2, depth - 1, sums, k);
  const double y = pw_combine(n - n2, depth - 1, sums, k);
  return x + y;
}
static double pw_sum_par(const double* w, const int64_t* perm, int64_t n, int depth) {
  std::vector<std::pair<int64_t, int64_t>> leaves;
  pw_leaves(0, n, depth, leaves);
  std::vector<double> sums(leaves.size());
  pool().run((int)leaves.size(), [&](int t) {
    sums[t] = pw_sum(w, perm + leaves[t].first, leaves[t].second);
  });
  size_t k = 0;
  return pw_combine(n, depth, sums.data(), k);
}
}  // namespace

extern "C" {

int skel_tree_build(const double* coords, int64_t n, int32_t dim, int64_t max_leaf, void** handle) {
  if (!coords || n < 1 || (dim != 2 && dim != 3) || max_leaf < 1 || !handle) return -1;
  Tree* T = nullptr;
  try {
    T = new Tree();
    build(*T, coords, n, dim, max_leaf);
  } catch (...) {          // bad_alloc (or a pool failure): no exception crosses the C ABI
    delete T;
    return -2;
  }
  if (T->nonfinite) {
    delete T;
    return -3;   // non-finite coordinate
  }
  // the neighbour lists of every cover are needed right after (the finest
  // level's first): start them now, overlapping the caller's node-array
  // copies and source setup; readers join first.  Failures on that thread
  // (or failing to start it) are absorbed: skel_tree_neighbors then builds
  // the lists itself and reports the error.
  try {
    T->nbr_thread = std::thread([T]() {
      try {
        all_neighbors(*T);
      } catch (...) {
        T->nbr_done = false;
      }
    });
  } catch (...) {
  }
  *handle = T;
  return 0;
}

int skel_tree_sizes(void* handle, int64_t* nnodes, int32_t* ncovers) {
  Tree* T = (Tree*)handle;
  if (!T) return -1;
  *nnodes = (int64_t)T->hw.size();
  *ncovers = (int32_t)T->covers.size();
  return 0;
}

int skel_tree_nodes(void* handle, double* center, double* hw, int64_t* lo, int64_t* hi,
                    int64_t* depth, int64_t* parent, int64_t* nchild, int64_t* perm) {
  Tree* T = (Tree*)handle;
  if (!T) return -1;
  const size_t nn = T->hw.size();
  if (center) std::memcpy(center, T->center.data(), nn * T->dim * sizeof(double));
  if (hw) std::memcpy(hw, T->hw.data(), nn * sizeof(double));
  if (lo) std::memcpy(lo, T->lo.data(), nn * sizeof(int64_t));
  if (hi) std::memcpy(hi, T->hi.data(), nn * sizeof(int64_t));
  if (depth) std::memcpy(depth, T->depth.data(), nn * sizeof(int64_t));
  if (parent) std::memcpy(parent, T->parent.data(), nn * sizeof(int64_t));
  if (nchild) std::memcpy(nchild, T->nchild.data(), nn * sizeof(int64_t));
  if (perm) std::memcpy(perm, T->perm.data(), T->n * sizeof(int64_t));
  return 0;
}

int skel_tree_perm_ptr(void* handle, const int64_t** perm) {
  Tree* T = (Tree*)handle;
  if (!T || !perm) return -1;
  *perm = T->perm.data();       // n entries, never written after the build, valid until skel_tree_free
  return 0;
}

int skel_tree_cover(void* handle, int32_t li, int64_t* count, int64_t* ids) {
  Tree* T = (Tree*)handle;
  if (!T || li < 0 || li >= (int32_t)T->covers.size()) return -1;
  *count = (int64_t)T->covers[li].size();
  if (ids) std::memcpy(ids, T->covers[li].data(), T->covers[li].size() * sizeof(int64_t));
  return 0;
}

int skel_tree_neighbors(void* handle, int32_t li, int64_t* off, int64_t* count, int64_t* idx) {
  Tree* T = (Tree*)handle;
  if (!T || li < 0 || li >= (int32_t)T->covers.size()) return -1;
  {
    std::lock_guard<std::mutex> l(T->nbr_m);
    if (T->nbr_thread.joinable()) T->nbr_thread.join();
  }
  try {
    all_neighbors(*T);
  } catch (...) {
    T->nbr_done = false;
    return -2;
  }
  *count = (int64_t)T->nbr_idx[li].size();
  if (off) std::memcpy(off, T->nbr_off[li].data(), T->nbr_off[li].size() * sizeof(int64_t));
  if (idx) std::memcpy(idx, T->nbr_idx[li].data(), T->nbr_idx[li].size() * sizeof(int64_t));
  return 0;
}

int skel_check_points(const double* coords, const double* normals, int64_t n, int32_t dim) {
  if (!coords || n < 1 || (dim != 2 && dim != 3)) return -1;
  const int T = pool().size();
  const int64_t chunk = (n + T - 1) / T;
  std::vector<char> bad_c(T, 0), bad_n(T, 0);
  pool().run(T, [&](int t) {
    const int64_t a0 = std::min(n, (int64_t)t * chunk), a1 = std::min(n, (int64_t)(t + 1) * chunk);
    bool bc = false, bn = false;
    for (int64_t i = a0; i < a1; ++i) {
      for (int a = 0; a < dim; ++a) bc |= !std::isfinite(coords[i * dim + a]);
      if (normals) {
        // |n| as np.linalg.norm(axis=1): squares, summed left to right, sqrt
        const double* v = normals + i * dim;
        double s = v[0] * v[0];
        for (int a = 1; a < dim; ++a) s = s + v[a] * v[a];
        bn |= std::fabs(std::sqrt(s) - 1.0) > 1e-12;   // NaN compares false, as in numpy
      }
    }
    bad_c[t] = bc;
    bad_n[t] = bn;
  });
  for (int t = 0; t < T; ++t)
    if (bad_c[t]) return -3;
  for (int t = 0; t < T; ++t)
    if (bad_n[t]) return -4;
  return 0;
}

int skel_perm_mean(const double* w, const int64_t* perm, int64_t n, double* out) {
  if (!w || !perm || !out || n < 1) return -1;
  *out = pw_sum_par(w, perm, n, 4) / (double)n;
  return 0;
}

int skel_tree_free(void* handle) {
  Tree* T = (Tree*)handle;
  if (T && T->nbr_thread.joinable()) T->nbr_thread.join();
  delete T;
  return 0;
}

}  // extern "C"
