// tree.cpp -- native host builder of the adaptive orthtree, its covers and the
// same-cover neighbour lists (K7).
//
// Restates geom.py:118-184 (centre splits, ties to the upper child, pruning,
// DFS node numbering and permutation, covers with early leaves repeated) and
// replaces level_neighbors (geom.py:205-219), which is O(p^2) in the
// reference, by an O(p) grid-hash candidate search followed by the identical
// predicate _boxes_touch (geom.py:187-189), so the lists are equal.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <utility>
#include <vector>

#include "../../include/skel_b200.h"

namespace {

struct Tree {
  int dim = 2;
  int64_t n = 0;
  std::vector<double> center;  // nnodes * dim
  std::vector<double> hw;
  std::vector<int64_t> lo, hi, depth, parent, nchild;
  std::vector<int64_t> perm;
  std::vector<std::vector<int64_t>> covers;  // finest first
  std::vector<std::vector<int64_t>> nbr_off, nbr_idx;  // per cover, lazily
  std::vector<char> nbr_done;
};

constexpr double kRootPad = 1e-12;
constexpr int kMaxDepth = 60;

struct Frame {
  std::vector<int64_t> idx;
  double c[3];
  double hw;
  int64_t depth;
  int64_t parent;
};

void build(Tree& T, const double* X, int64_t n, int d, int64_t max_leaf) {
  T.dim = d;
  T.n = n;
  double lo_c[3], hi_c[3], c0[3];
  for (int a = 0; a < d; ++a) {
    lo_c[a] = INFINITY;
    hi_c[a] = -INFINITY;
  }
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < d; ++a) {
      double v = X[i * d + a];
      lo_c[a] = std::min(lo_c[a], v);
      hi_c[a] = std::max(hi_c[a], v);
    }
  double ext = 0.0, cabs = 0.0;
  for (int a = 0; a < d; ++a) {
    c0[a] = 0.5 * (lo_c[a] + hi_c[a]);
    ext = std::max(ext, hi_c[a] - lo_c[a]);
    cabs = std::max(cabs, std::fabs(c0[a]));
  }
  double hw0 = 0.5 * ext;
  double scale = std::max(std::max(hw0, cabs), 1.0);
  hw0 = hw0 * (1.0 + kRootPad) + kRootPad * scale;

  T.perm.assign(n, 0);
  int64_t cursor = 0;
  std::vector<Frame> stack;
  Frame root;
  root.idx.resize(n);
  for (int64_t i = 0; i < n; ++i) root.idx[i] = i;
  for (int a = 0; a < d; ++a) root.c[a] = c0[a];
  root.hw = hw0;
  root.depth = 0;
  root.parent = -1;
  stack.push_back(std::move(root));
  const int nkids = 1 << d;
  while (!stack.empty()) {
    Frame f = std::move(stack.back());
    stack.pop_back();
    const int64_t me = (int64_t)T.hw.size();
    for (int a = 0; a < d; ++a) T.center.push_back(f.c[a]);
    T.hw.push_back(f.hw);
    T.lo.push_back(cursor);
    T.hi.push_back(cursor + (int64_t)f.idx.size());
    T.depth.push_back(f.depth);
    T.parent.push_back(f.parent);
    T.nchild.push_back(0);
    if (f.parent >= 0) T.nchild[f.parent] += 1;
    const int64_t sz = (int64_t)f.idx.size();
    if (sz <= max_leaf || f.depth >= kMaxDepth) {
      for (int64_t t = 0; t < sz; ++t) T.perm[cursor + t] = f.idx[t];
      cursor += sz;
      continue;
    }
    std::vector<std::vector<int64_t>> parts(nkids);
    for (int64_t t = 0; t < sz; ++t) {
      const int64_t i = f.idx[t];
      int code = 0;
      for (int a = 0; a < d; ++a) code |= (X[i * d + a] >= f.c[a] ? 1 : 0) << a;
      parts[code].push_back(i);
    }
    std::vector<Frame> kids;
    for (int c = 0; c < nkids; ++c) {
      if (parts[c].empty()) continue;
      Frame k;
      k.idx = std::move(parts[c]);
      for (int a = 0; a < d; ++a) k.c[a] = f.c[a] + (((c >> a) & 1) ? 0.5 : -0.5) * f.hw;
      k.hw = 0.5 * f.hw;
      k.depth = f.depth + 1;
      k.parent = me;
      kids.push_back(std::move(k));
    }
    for (auto it = kids.rbegin(); it != kids.rend(); ++it) stack.push_back(std::move(*it));
  }
  const int64_t nn = (int64_t)T.hw.size();
  int64_t maxd = 0;
  for (int64_t i = 0; i < nn; ++i) maxd = std::max(maxd, T.depth[i]);
  for (int64_t f = maxd; f >= 0; --f) {
    std::vector<int64_t> cov;
    for (int64_t i = 0; i < nn; ++i)
      if (T.depth[i] == f || (T.nchild[i] == 0 && T.depth[i] < f)) cov.push_back(i);
    std::stable_sort(cov.begin(), cov.end(),
                     [&](int64_t x, int64_t y) { return T.lo[x] < T.lo[y]; });
    T.covers.push_back(std::move(cov));
  }
  T.nbr_off.resize(T.covers.size());
  T.nbr_idx.resize(T.covers.size());
  T.nbr_done.assign(T.covers.size(), 0);
}

void neighbors(Tree& T, int li) {
  if (T.nbr_done[li]) return;
  const std::vector<int64_t>& ids = T.covers[li];
  const int64_t p = (int64_t)ids.size();
  const int d = T.dim;
  std::vector<int64_t>& off = T.nbr_off[li];
  std::vector<int64_t>& idx = T.nbr_idx[li];
  off.assign(p + 1, 0);
  idx.clear();
  T.nbr_done[li] = 1;
  if (p < 2) return;
  const double tol = 1e-9 * T.hw[0];
  double hmin = INFINITY;
  for (int64_t a = 0; a < p; ++a) hmin = std::min(hmin, T.hw[ids[a]]);
  const double cell = 2.0 * hmin;
  double origin[3];
  for (int a = 0; a < d; ++a) origin[a] = T.center[a] - T.hw[0] - 2.0 * cell;
  std::vector<int64_t> clo(p * d), chi(p * d);
  int64_t gdim = 1;
  for (int64_t b = 0; b < p; ++b) {
    const int64_t nd = ids[b];
    for (int a = 0; a < d; ++a) {
      const double c = T.center[nd * d + a], h = T.hw[nd];
      clo[b * d + a] = (int64_t)std::floor((c - h - tol - origin[a]) / cell);
      chi[b * d + a] = (int64_t)std::floor((c + h + tol - origin[a]) / cell);
      gdim = std::max(gdim, chi[b * d + a] + 2);
    }
  }
  // (cell key, box) registrations
  std::vector<std::pair<int64_t, int64_t>> reg;
  for (int64_t b = 0; b < p; ++b) {
    int64_t span[3] = {1, 1, 1}, tot = 1;
    for (int a = 0; a < d; ++a) {
      span[a] = chi[b * d + a] - clo[b * d + a] + 1;
      tot *= span[a];
    }
    for (int64_t t = 0; t < tot; ++t) {
      int64_t rem = t, key = 0;
      for (int a = 0; a < d; ++a) {
        key = key * gdim + clo[b * d + a] + rem % span[a];
        rem /= span[a];
      }
      reg.emplace_back(key, b);
    }
  }
  std::sort(reg.begin(), reg.end());
  std::vector<std::pair<int64_t, int64_t>> pairs;
  size_t s = 0;
  while (s < reg.size()) {
    size_t e = s;
    while (e < reg.size() && reg[e].first == reg[s].first) ++e;
    for (size_t u = s; u < e; ++u)
      for (size_t v = u + 1; v < e; ++v) pairs.emplace_back(reg[u].second, reg[v].second);
    s = e;
  }
  std::sort(pairs.begin(), pairs.end());
  pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
  std::vector<std::pair<int64_t, int64_t>> adj;
  for (auto& pr : pairs) {
    const int64_t na = ids[pr.first], nb = ids[pr.second];
    bool touch = true;
    for (int a = 0; a < d && touch; ++a) {
      double gap = std::fabs(T.center[na * d + a] - T.center[nb * d + a]) - (T.hw[na] + T.hw[nb]);
      touch = gap <= tol;
    }
    if (touch) {
      adj.emplace_back(pr.first, pr.second);
      adj.emplace_back(pr.second, pr.first);
    }
  }
  std::sort(adj.begin(), adj.end());
  idx.resize(adj.size());
  for (size_t t = 0; t < adj.size(); ++t) {
    off[adj[t].first + 1] += 1;
    idx[t] = adj[t].second;
  }
  for (int64_t b = 0; b < p; ++b) off[b + 1] += off[b];
}

}  // namespace

extern "C" {

int skel_tree_build(const double* coords, int64_t n, int32_t dim, int64_t max_leaf, void** handle) {
  if (!coords || n < 1 || (dim != 2 && dim != 3) || max_leaf < 1 || !handle) return -1;
  Tree* T = new Tree();
  build(*T, coords, n, dim, max_leaf);
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
  neighbors(*T, li);
  *count = (int64_t)T->nbr_idx[li].size();
  if (off) std::memcpy(off, T->nbr_off[li].data(), T->nbr_off[li].size() * sizeof(int64_t));
  if (idx) std::memcpy(idx, T->nbr_idx[li].data(), T->nbr_idx[li].size() * sizeof(int64_t));
  return 0;
}

int skel_tree_free(void* handle) {
  delete (Tree*)handle;
  return 0;
}

}  // extern "C"
