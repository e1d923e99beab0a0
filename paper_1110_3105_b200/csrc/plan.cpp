// plan.cpp -- host-side per-level bookkeeping of the compression sweep and
// the factorization (the numpy index arithmetic of skel.compress_source /
// solver.FactorRun.add_level in one native pass per level): dof and slab
// offsets, target heights, size classes, the big-box selection and the
// size-bucketed launch orders.  Single-threaded: one pass over p boxes plus
// the neighbour lists; the Python version spent ~5 ms per 30k-box level.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

#include "../../include/skel_b200.h"

namespace {

inline int64_t al16(int64_t v) { return (v + 15) / 16 * 16; }

// host mirror of level_smem_fixed<T> (csrc/id_level.cu), an upper bound
inline int64_t level_smem_fixed(int64_t max_n) {
  const int64_t sh = al16(96 + 8 * 32 + 4 * 32);
  const int64_t hdr = al16(4 * (257 + 256 + 9 + 9 + 2) + 8 * 32 + 8);
  return sh + hdr + al16(80 * max_n) + al16(24 * max_n) + al16(8 * max_n) + al16(48 * max_n);
}

inline int64_t lower_bound_idx(const int64_t* a, int n, int64_t v) {
  return std::lower_bound(a, a + n, v) - a;     // np.searchsorted(side="left")
}

// group boxes by class (cls >= 0), each group by descending key, ties by
// position; writes order[], bucket starts (nb + 1); returns nb
int buckets_by_class(int64_t p, const int64_t* cls, const int64_t* key, int32_t* order,
                     int32_t* bstart) {
  // counting sort by class (stable), then each class by descending key with
  // ties by position: sort (key, position) pairs packed into one integer
  int64_t cmax = -1;
  for (int64_t a = 0; a < p; ++a) cmax = std::max(cmax, cls[a]);
  if (cmax < 0) {
    bstart[0] = 0;
    return 0;
  }
  std::vector<int64_t> cnt(cmax + 2, 0);
  for (int64_t a = 0; a < p; ++a)
    if (cls[a] >= 0) cnt[cls[a] + 1]++;
  for (int64_t c = 0; c <= cmax; ++c) cnt[c + 1] += cnt[c];
  std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
  for (int64_t a = 0; a < p; ++a)
    if (cls[a] >= 0) order[pos[cls[a]]++] = (int32_t)a;
  int nb = 0;
  // within a class: descending key, ties by position.  `order` is in position
  // order already (stable counting sort above), so a stable LSD radix sort on
  // d = kmax - key gives exactly that order (a comparison sort of the 30k-box
  // finest levels cost ~1 ms of GPU-idle host time per level)
  std::vector<uint32_t> d, d2;
  std::vector<int32_t> o2;
  for (int64_t c = 0; c <= cmax; ++c) {
    const int64_t s = cnt[c], e = cnt[c + 1];
    if (e == s) continue;
    bstart[nb++] = (int32_t)s;
    const int64_t m = e - s;
    if (key && m > 1) {
      int64_t kmax = key[order[s]], kmin = kmax;
      for (int64_t i = s; i < e; ++i) {
        kmax = std::max(kmax, key[order[i]]);
        kmin = std::min(kmin, key[order[i]]);
      }
      const uint64_t span = (uint64_t)(kmax - kmin);
      if (span == 0) continue;
      if (span >> 32) {                       // huge keys: comparison sort
        std::vector<uint64_t> tmp(m);
        std::stable_sort(order + s, order + e,
                         [&](int32_t a, int32_t b) { return key[a] > key[b]; });
        continue;
      }
      d.resize(m); d2.resize(m); o2.resize(m);
      for (int64_t i = 0; i < m; ++i) d[i] = (uint32_t)(kmax - key[order[s + i]]);
      int32_t* oa = order + s;
      int32_t* ob = o2.data();
      uint32_t* da = d.data();
      uint32_t* db = d2.data();
      for (int shift = 0; shift < 32 && (span >> shift); shift += 11) {
        int64_t hist[2049] = {0};
        for (int64_t i = 0; i < m; ++i) hist[((da[i] >> shift) & 2047u) + 1]++;
        for (int b = 0; b < 2048; ++b) hist[b + 1] += hist[b];
        for (int64_t i = 0; i < m; ++i) {
          const int64_t q = hist[(da[i] >> shift) & 2047u]++;
          ob[q] = oa[i];
          db[q] = da[i];
        }
        std::swap(oa, ob);
        std::swap(da, db);
      }
      if (oa != order + s) std::memcpy(order + s, oa, sizeof(int32_t) * m);
    }
  }
  bstart[nb] = (int32_t)cnt[cmax + 1];
  return nb;
}

}  // namespace

extern "C" {

int skel_plan_id_level(int64_t p, const int64_t* nr, const int64_t* nc, const int64_t* noff,
                       const int64_t* nidx, const int64_t* neff, const uint8_t* own, int32_t elem,
                       int64_t optin, const int64_t* wcls, int32_t n_wcls, const int64_t* mcls,
                       int32_t n_mcls, int64_t big_n, int64_t rand_cut, int64_t small_level,
                       int64_t* rdof_off, int64_t* cdof_off, int64_t* m0, int64_t* m1,
                       int64_t* d_off, int64_t* l_off, int64_t* r_off, int64_t* need_m,
                       int64_t* need_n, uint8_t* big, int32_t* order, int32_t* bstart,
                       int32_t* nbuckets, int64_t* merged) {
  std::vector<int64_t> cls(p), wb(p);
  rdof_off[0] = cdof_off[0] = d_off[0] = l_off[0] = r_off[0] = 0;
  bool any_fit = false;
  int64_t fm = 0, fn = 0, fw = 0;
  for (int64_t a = 0; a < p; ++a) {
    const int64_t r = nr[a], c = nc[a], o = own ? own[a] : 1;
    rdof_off[a + 1] = rdof_off[a] + r;
    cdof_off[a + 1] = cdof_off[a] + c;
    d_off[a + 1] = d_off[a] + r * c * o;
    l_off[a + 1] = l_off[a] + r * r * o;
    r_off[a + 1] = r_off[a] + c * c * o;
    int64_t s0 = 0, s1 = 0;
    for (int64_t e = noff[a]; e < noff[a + 1]; ++e) {
      const int64_t b = nidx[e];
      s0 += nc[b];
      s1 += nr[b];
    }
    m0[a] = s0 + neff[a];
    m1[a] = s1 + neff[a];
    need_m[a] = std::max(m0[a], m1[a]);
    if (elem == 8) need_m[a] = (need_m[a] + 1) & ~int64_t(1);   // even ld, real CPQR tile
    need_n[a] = std::max<int64_t>(std::max(r, c), 1);
    wb[a] = need_m[a] * need_n[a] * elem;
    const int64_t fixed = level_smem_fixed(need_n[a]);
    // big: the reference's randomized-ID selector (skel.py:419-421) on
    // either side, too wide, or a target that cannot fit one CTA
    const bool rnd = m0[a] > std::max(rand_cut, 4 * r + 256) || m1[a] > std::max(rand_cut, 4 * c + 256);
    const bool bg = rnd || need_n[a] > big_n || fixed > optin;
    big[a] = (uint8_t)(o && bg);
    cls[a] = (o && !bg) ? lower_bound_idx(wcls, n_wcls, wb[a]) * 16 + lower_bound_idx(mcls, n_mcls, need_m[a])
                        : -1;
    if ((!bg || !o) && fixed + wb[a] <= optin) {
      any_fit = true;
      fm = std::max(fm, need_m[a]);
      fn = std::max(fn, need_n[a]);
      fw = std::max(fw, need_m[a] * need_n[a]);
    }
  }
  merged[0] = 0;
  if (p <= small_level && any_fit && level_smem_fixed(fn) + fw * elem <= optin) {
    // few boxes: one launch for all that fit, configured over the whole level
    bool first = false;
    for (int64_t a = 0; a < p; ++a) {
      const bool fits = cls[a] >= 0 && level_smem_fixed(need_n[a]) + wb[a] <= optin;
      first |= fits;
      cls[a] = fits ? 0 : (cls[a] >= 0 ? cls[a] + 1 : -1);
    }
    merged[0] = first ? 2 : 1;     // 2: bucket 0 holds the merged boxes
    merged[1] = fm;
    merged[2] = fn;
    merged[3] = fw;
  }
  *nbuckets = buckets_by_class(p, cls.data(), wb.data(), order, bstart);
  return 0;
}

int skel_plan_factor_level(int64_t p, const int64_t* nr, const int64_t* nc, const int64_t* kr,
                           const int64_t* kc, const uint8_t* own, int32_t elem, int64_t optin,
                           const int64_t* fcls, int32_t n_fcls, int64_t big_n, int64_t small_level,
                           const int64_t* scls, int32_t n_scls, int64_t* n, int64_t* k,
                           uint8_t* sq_bad, uint8_t* lam_bad, int64_t* dd_off, int64_t* ld_off,
                           int64_t* lam_off, int64_t* noff, int64_t* koff, uint8_t* big,
                           int32_t* order, int32_t* bstart, int32_t* nbuckets, int32_t* sorder,
                           int32_t* sstart, int32_t* nsbuckets, int64_t* merged) {
  std::vector<int64_t> cls(p), need(p), sc(p);
  dd_off[0] = ld_off[0] = lam_off[0] = noff[0] = koff[0] = 0;
  bool any_fit = false;
  int64_t fn = 0, fk = 0;
  for (int64_t a = 0; a < p; ++a) {
    const bool sq = nr[a] != nc[a];
    const bool lb = !sq && nr[a] > 0 && kr[a] != kc[a];
    sq_bad[a] = sq;
    lam_bad[a] = lb;
    n[a] = (sq || lb) ? 0 : nr[a];
    k[a] = n[a] > 0 ? kr[a] : 0;
    const int64_t o = own ? own[a] : 1;
    const int64_t no = n[a] * o;
    dd_off[a + 1] = dd_off[a] + no * no;
    ld_off[a + 1] = ld_off[a] + no * k[a];
    lam_off[a + 1] = lam_off[a] + k[a] * k[a];
    noff[a + 1] = noff[a] + n[a];
    koff[a + 1] = koff[a] + k[a];
    need[a] = (n[a] * n[a] + 4 * n[a] * k[a] + k[a] * k[a] + 4 * n[a] + k[a]) * elem;   // fac_elems (factor.cu)
    const bool bg = no >= big_n;
    big[a] = (uint8_t)(no > 0 && bg);
    cls[a] = (no > 0 && !bg) ? lower_bound_idx(fcls, n_fcls, need[a]) : -1;
    sc[a] = no > 0 ? lower_bound_idx(scls, n_scls, n[a]) : -1;
    if (n[a] > 0 && n[a] < big_n && need[a] + 1024 + 4 * n[a] <= optin) {
      any_fit = true;
      fn = std::max(fn, n[a]);
      fk = std::max(fk, k[a]);
    }
  }
  merged[0] = 0;
  if (p <= small_level && any_fit &&
      (fn * fn + 4 * fn * fk + fk * fk + 4 * fn + fk) * elem + 1024 + 4 * fn <= optin) {
    bool first = false;
    for (int64_t a = 0; a < p; ++a) {
      const bool fits = cls[a] >= 0 && need[a] + 1024 + 4 * n[a] <= optin;
      first |= fits;
      cls[a] = fits ? 0 : (cls[a] >= 0 ? cls[a] + 1 : -1);
    }
    merged[0] = first ? 2 : 1;     // 2: bucket 0 holds the merged boxes
    merged[1] = fn;
    merged[2] = fk;
  }
  *nbuckets = buckets_by_class(p, cls.data(), need.data(), order, bstart);
  *nsbuckets = buckets_by_class(p, sc.data(), nullptr, sorder, sstart);
  return 0;
}

}  // extern "C"
