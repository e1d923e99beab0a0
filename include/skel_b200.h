/*
 * skel_b200.h -- C ABI of libskel_sm100.so, the B200 (sm_100a) engine behind
 * the recursive-skeletonization factor / multi-RHS solve path.
 *
 * Plain C types only (no torch types): device buffers are raw pointers owned
 * by the caller, streams are passed as void* (cudaStream_t), every call is
 * stream-ordered and returns an int status (0 = ok, >0 = CUDA error code,
 * <0 = invalid argument).  Per-box numerical outcomes come back in status
 * arrays and are mapped to the reference's exceptions / warnings by the host
 * package (paper_1110_3105_b200).
 *
 * Each entry point names the reference interface (skelkit 0.1.0, file:line)
 * whose work it replaces.
 */
#ifndef SKEL_B200_H
#define SKEL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- matrix sources (the matrix-source protocol, skel.py:289-290) ------- */

enum {
  SKEL_EQ_LAPLACE = 0,
  SKEL_EQ_HELMHOLTZ = 1
};
enum {
  SKEL_LAYER_SINGLE = 0,
  SKEL_LAYER_DOUBLE = 1
};
enum {
  /* BieSystem in tree order (bie.py:135-176, bie.py:233-262): double layer
     of `equation`, curvature-limit (Laplace) / zero (Helmholtz) diagonal,
     optional KR10, + identity_coef on the diagonal; single-layer proxies,
     row proxies scaled by wscale. */
  SKEL_SRC_BIE = 0,
  /* KernelSource (skel.py:100-124) + optional `diag` on coincident indices */
  SKEL_SRC_KERNEL = 1,
  /* combined field (D_k - i k S_k) * KR10 + identity_coef (BASELINE config 3) */
  SKEL_SRC_CFIE = 2,
  /* sound-hard multiple scattering (bie.py:305-367): target-normal derivative
     of the 2D Helmholtz single layer, -(ik/4) H1(kr) (x-y).nu_x / r * w_y,
     KR10 within a scatterer, + identity_coef (-1/2) on the diagonal; row
     proxies = the same Neumann trace of the proxy field (unweighted), column
     proxies = single layer * w */
  SKEL_SRC_NTRACE = 3
};

typedef struct {
  /* geometry in TREE order, device pointers, SoA */
  const double* x;
  const double* y;
  const double* z;        /* NULL in 2D */
  const double* nx;       /* normals; NULL unless a double layer is used */
  const double* ny;
  const double* nz;
  const double* w;        /* quadrature weights; NULL = unweighted */
  const double* curv;     /* curvature (2D Laplace curvature limit) */
  const int64_t* orig;    /* tree position -> original index */
  int64_t n;
  int32_t dim;
  int32_t kind;           /* SKEL_SRC_* */
  int32_t equation;       /* SKEL_EQ_* */
  int32_t layer;          /* SKEL_LAYER_* (KERNEL kind) */
  int32_t curvature_limit;/* 1: coincident DL entries = -kappa/(4 pi) */
  int32_t kr10;           /* 1: Kapur-Rokhlin order-10 reweighting */
  double k;               /* wavenumber */
  double identity_coef;   /* added where row == col (BIE / CFIE) */
  double diag;            /* added where row == col (KERNEL) */
  double wscale;          /* row-proxy scale (bie.py:251); 1 otherwise */
  double coincide_tol;    /* r < coincide_tol counts as coincident */
  /* optional point groups (several scatterers in one source): KR10 applies
     only within a group, on local indices (orig - grp_start[g]) cyclic in
     grp_size[g]; NULL = one group of size n */
  const int32_t* grp;     /* per ORIGINAL index */
  const int64_t* grp_start;
  const int64_t* grp_size;
} SkelSource;

/* ---- one cover (tree level) of the compression sweep -------------------- */

typedef struct {
  int32_t nbox;
  int32_t level;             /* li (0 = finest) */
  int32_t equalize;          /* equalize_ranks (skel.py:377-382) */
  int32_t n_unit;            /* rows in the unit-proxy table */
  double eps;
  /* dof lists: CSR over boxes, tree positions (int32) */
  const int64_t* rdof_off;   /* nbox+1 */
  const int32_t* rdofs;
  const int64_t* cdof_off;
  const int32_t* cdofs;
  /* children: box a's children are the previous cover's positions
     [child_off[a], child_off[a+1]) (contiguous, skel.py:252-264); their
     ranks give the children's diagonal sub-blocks of D (skel.py:345-348).
     All three are NULL at li = 0. */
  const int64_t* child_off;  /* nbox+1 */
  const int32_t* prev_kr;
  const int32_t* prev_kc;
  /* neighbours in this cover (ascending), CSR */
  const int64_t* nbr_off;
  const int32_t* nbr;
  /* proxy surface: centre (nbox*dim), radius, and which unit table rows */
  const double* box_c;
  const double* box_r;
  const int32_t* pxy_begin;  /* first row of this box's unit table */
  const int32_t* pxy_count;  /* n_eff */
  const double* pxy_unit;    /* n_unit * dim unit points */
  /* outputs (capacity slabs; offsets are element offsets) */
  const int64_t* d_off;      /* D: nr x nc row-major */
  const int64_t* l_off;      /* L: nr x kr row-major, capacity nr*nr */
  const int64_t* r_off;      /* R: kc x nc row-major, capacity nc*nc */
  void* D;
  void* L;
  void* R;
  int32_t* rskel;            /* sorted row skeleton tree positions, at rdof_off */
  int32_t* cskel;
  int32_t* kr;               /* per box ranks */
  int32_t* kc;
  int32_t* flags;            /* bit0/1: |P| > 2 (row/col); bit2: ranks differ */
  void* scratch;             /* global fallback for targets over the smem limit */
  int64_t scratch_bytes;
  int32_t debug_skip;        /* developer timing only: 1 = assembly only, 2 = + norms */
} SkelLevel;

/* Assemble + ID + equalize every box of one cover, both sides.
 * Replaces build_node (skel.py:341-391): D = A(rd,cd) with children blocks
 * zeroed, proxy-compressed targets t_row.T / t_col (skel.py:349-368),
 * id_fixed_precision x2 (lowrank.py:48-161), equalize (skel.py:377-382),
 * skeleton sort and L/R (skel.py:384-391).  `box_order` lists the boxes to
 * process (sorted by size by the caller); `max_m`/`max_n` bound the target
 * height / width and `max_w` its m*n element count over the listed boxes.
 * field: 0 = float64, 1 = complex128. */
int skel_id_level(const SkelSource* src, const SkelLevel* lv, const int32_t* box_order,
                  int32_t nbox_run, int32_t max_m, int32_t max_n, int64_t max_w,
                  int32_t field, void* stream);

/* D = A(rd, cd) of every box of a cover with the children's diagonal
 * blocks zeroed (skel.py:344-348), into lv->D at lv->d_off.  order (nrun
 * box indices) restricts the launch to a subset (a rank's own boxes); NULL
 * = all lv->nbox boxes.  max_n bounds n_r and n_c. */
int skel_assemble_D(const SkelSource* src, const SkelLevel* lv, const int32_t* order, int32_t nrun,
                    int32_t max_n, int32_t field, void* stream);

/* Dense top-level skeleton matrix S = A(row_skel_a, col_skel_b), a != b,
 * zero diagonal blocks (skel.py:399-408). rows/cols: tree positions; rbox/cbox:
 * owning box of each row/col. S is K_r x K_c row-major. */
int skel_assemble_S(const SkelSource* src, const int32_t* rows, const int32_t* rbox,
                    int32_t Kr, const int32_t* cols, const int32_t* cbox, int32_t Kc,
                    void* S, int32_t field, void* stream);

/* Dense block A(rows, cols) (BieSystem.block / KernelSource.block / eval_block,
 * kernels.py:82-161, bie.py:158-172), row-major m x n. */
int skel_eval_block(const SkelSource* src, const int32_t* rows, int32_t m,
                    const int32_t* cols, int32_t n, void* out, int32_t field,
                    void* stream);

/* Batched column ID of explicit matrices (id_fixed_precision,
 * lowrank.py:136-161).  Matrix b is column-major m[b] x n[b] at a_off[b].
 * Outputs: rank[b], skel (pivot order, n[b] capacity at skel_off[b]),
 * proj (rank x n row-major, capacity n*n at proj_off[b]), bigP[b] = max|P|,
 * ratio[b] (nullable) = the first rejected pivot norm over the leading one
 * (InterpDecomp.achieved_error, lowrank.py:116-118,161; 0 when the CPQR ran
 * to min(m, n) or hit an exactly zero pivot). */
int skel_id_batched(const void* A, const int64_t* a_off, const int32_t* m,
                    const int32_t* n, int32_t nmat, double eps,
                    const int32_t* min_rank, int32_t* rank, int32_t* skel,
                    const int64_t* skel_off, void* proj, const int64_t* proj_off,
                    double* bigP, double* ratio, int32_t field, void* scratch,
                    int64_t scratch_bytes, int32_t max_m, int32_t max_n,
                    void* stream);

/* pivoted_qr (lowrank.py:48-119) for a batch: the same CPQR as skel_id_batched,
 * returning per matrix the WHOLE pivot permutation (piv: n[b] entries at
 * piv_off[b]), rank[b] = the completed CPQR steps (no min_rank padding), and
 * the rank x n upper-trapezoidal factor R with its columns in pivot order
 * (row-major at rfac_off[b]; capacity min(m,n) x n).  proj / bigP / ratio as
 * for skel_id_batched (proj capacity n x n per matrix). */
int skel_pivoted_qr_batched(const void* A, const int64_t* a_off, const int32_t* m,
                            const int32_t* n, int32_t nmat, double eps,
                            const int32_t* min_rank, int32_t* rank, int32_t* piv,
                            const int64_t* piv_off, void* rfac, const int64_t* rfac_off,
                            void* proj, const int64_t* proj_off, double* bigP,
                            double* ratio, int32_t field, void* scratch,
                            int64_t scratch_bytes, int32_t max_m, int32_t max_n,
                            void* stream);

/* ---- telescoping factorization (solver.py:187-276) --------------------- */

typedef struct {
  int32_t nbox;
  int32_t level;
  double regularize;
  /* per box sizes: n (=nr=nc), k (=kr=kc) */
  const int32_t* n;
  const int32_t* k;
  /* compressed inputs (capacity slabs of SkelLevel) */
  const int64_t* d_off;
  const int64_t* l_off;
  const int64_t* r_off;
  const void* D;
  const void* L;
  const void* R;
  /* children Lambda of the previous level: per box child range into the
     previous level's lam_off (NULL at the finest level) */
  const int64_t* child_off;
  const int64_t* prev_lam_off;
  const void* prev_lam;
  const int32_t* prev_k;
  /* outputs, tight slabs */
  const int64_t* dd_off;     /* n*n */
  const int64_t* ld_off;     /* n*k */
  const int64_t* rd_off;     /* k*n */
  const int64_t* lam_off;    /* k*k */
  void* Dd;
  void* Ld;
  void* Rd;
  void* Lam;
  int32_t* status;           /* 0 ok, 1 zero pivot in D, 2 zero pivot in Lambda */
  double* rcond_d;
  double* rcond_m;
  void* scratch;
  int64_t scratch_bytes;
  /* optional subset: process boxes order[0..nrun) (NULL: all nbox boxes) */
  const int32_t* order;
  int32_t nrun;
} SkelFactorLevel;

/* factor_node over every box of one level (solver.py:224-262). */
int skel_factor_level(const SkelFactorLevel* fl, int32_t max_n, int32_t max_k,
                      int32_t field, void* stream);

/* Invert a dense K x K matrix (row-major) with partial pivoting in place,
 * plus the pivoted LU copy (solver.py:269-274 `_lu(Shat)`).  status: 0 ok,
 * 1 zero pivot.  rcond (1-norm) written to *rcond. */
int skel_dense_inverse(void* A, void* lu, int32_t* ipiv, int32_t K, double regularize,
                       int32_t* status, double* rcond, int32_t field, void* scratch,
                       void* stream);

/* out[2i], out[2i+1] = Re, Im of H0^(1)(z[i]) = J0 + i Y0 (kernels.py:65-75). */
int skel_bessel_h0(const double* z, int64_t n, double* out, void* stream);

/* ---- host planning of one level (csrc/plan.cpp) --------------------------
 * The index bookkeeping of compress_source / factor per level in one native
 * pass: dof / slab offsets, target heights (sum of neighbour dofs + proxies),
 * size classes, big-box selection (randomized-ID selector skel.py:419-421,
 * width, shared-memory fit), size-bucketed launch orders (class ascending,
 * size descending).  `merged` = {flag, max_m, max_n, max_w} (ID) or
 * {flag, max_n, max_k} (factor): levels with <= small_level boxes launch
 * every fitting box at once, configured over the whole level. */
int skel_plan_id_level(int64_t p, const int64_t* nr, const int64_t* nc, const int64_t* noff,
                       const int64_t* nidx, const int64_t* neff, const uint8_t* own, int32_t elem,
                       int64_t optin, const int64_t* wcls, int32_t n_wcls, const int64_t* mcls,
                       int32_t n_mcls, int64_t big_n, int64_t rand_cut, int64_t small_level,
                       int64_t* rdof_off, int64_t* cdof_off, int64_t* m0, int64_t* m1,
                       int64_t* d_off, int64_t* l_off, int64_t* r_off, int64_t* need_m,
                       int64_t* need_n, uint8_t* big, int32_t* order, int32_t* bstart,
                       int32_t* nbuckets, int64_t* merged);
int skel_plan_factor_level(int64_t p, const int64_t* nr, const int64_t* nc, const int64_t* kr,
                           const int64_t* kc, const uint8_t* own, int32_t elem, int64_t optin,
                           const int64_t* fcls, int32_t n_fcls, int64_t big_n, int64_t small_level,
                           const int64_t* scls, int32_t n_scls, int64_t* n, int64_t* k,
                           uint8_t* sq_bad, uint8_t* lam_bad, int64_t* dd_off, int64_t* ld_off,
                           int64_t* lam_off, int64_t* noff, int64_t* koff, uint8_t* big,
                           int32_t* order, int32_t* bstart, int32_t* nbuckets, int32_t* sorder,
                           int32_t* sstart, int32_t* nsbuckets, int64_t* merged);

/* ---- big boxes (one box over the whole GPU; csrc/big.cu) ---------------
 * Used for boxes whose target does not fit a per-box CTA (3D coarse levels)
 * and for every target the reference sends to id_randomized
 * (m > max(4096, 4n + 256), skel.py:419-421). */

/* bytes of the CPQR state buffer for n columns */
int64_t skel_big_state_bytes(int32_t n);

/* Target of box `box`, side 0 = t_row.T, 1 = t_col (skel.py:349-368), into W
 * (m x n column-major, leading dimension ld).  nbr_box / nbr_pref (device):
 * the box's neighbours and the prefix sums of their dof counts (nnb + 1). */
int skel_big_target(const SkelSource* src, const SkelLevel* lv, int32_t box, int32_t side,
                    const int32_t* nbr_box, const int32_t* nbr_pref, int32_t nnb, int32_t m,
                    int32_t n, void* W, int64_t ld, int32_t field, void* stream);

/* Cooperative CPQR of W in place (pivoted_qr, lowrank.py:48-119).  resume
 * bit 0: continue from the state's rank with the new min_rank; bit 1
 * (equalisation, skel.py:377-382): stop after exactly min_rank steps, so the
 * box stays square even where a recomputed stale norm would carry the
 * reference's re-run past k. */
int skel_cpqr_big(void* W, int32_t m, int32_t n, int64_t ld, double eps, int32_t min_rank,
                  int32_t resume, void* state, int32_t field, void* stream);

/* P = R11^-1 R12 in place + padding to min_rank (lowrank.py:122-161). */
int skel_big_interp(void* W, int32_t n, int64_t ld, void* state, int32_t min_rank, int32_t field,
                    void* stream);

/* Sorted skeletons, L or R, kr / kc and the |P| > 2 flag of box `box`. */
int skel_big_output(const SkelLevel* lv, int32_t box, int32_t side, const void* W, int64_t ld,
                    const void* state, int32_t n, int32_t field, void* stream);

/* Y (m x n) = X^T A; X k x m, A k x n; column-major (the sketch Omega A). */
int skel_gemm_tn(int32_t m, int32_t n, int32_t k, const void* X, int64_t ldx, const void* A,
                 int64_t lda, void* Y, int64_t ldy, int32_t field, void* stream);

/* y = A x (trans 0) or A^H x (trans 1); A m x n column-major. */
int skel_gemv(int32_t trans, int32_t m, int32_t n, const void* A, int64_t lda, const void* x,
              void* y, int32_t field, void* stream);

/* Probe of id_randomized (lowrank.py:220-228): u = P v, z = A v - A[:, skel] u
 * for the sketch's CPQR state (interp already applied to Ysk). */
int skel_big_probe(int32_t m, int32_t n, const void* A, int64_t lda, const void* Ysk, int64_t ldy,
                   const void* state, const void* v, void* u, void* z, int32_t field, void* stream);

/* Cooperative Gauss-Jordan inverse (partial pivoting) of a big n x n
 * row-major matrix in place; *status (zeroed by the caller) = 1 on an exact
 * zero pivot.  scratch: skel_gj_scratch_bytes(n). */
int64_t skel_gj_scratch_bytes(int32_t n);

/* LU with partial pivoting in place (getrf conventions: unit-lower L, U,
 * 0-based piv as scipy.linalg.lu_factor; the reference's Shat factorization,
 * solver.py:269-274, and the factored container's S_lu).  *status (zeroed by
 * the caller) = 1 on an exact zero pivot.  scratch: skel_gj_scratch_bytes(n). */
int skel_dense_lu(void* A, int32_t n, int32_t* piv, int32_t* status, int32_t field, void* scratch,
                  void* stream);

/* inv = A^-1 (row-major) from skel_dense_lu factors (getrs order per column). */
int skel_lu_inverse(const void* lu, const int32_t* piv, int32_t n, void* inv, int32_t field,
                    void* stream);

/* factor_node of ONE big box (n = nr = nc, k) over the whole GPU: cooperative
 * inverses of D_eff and M = R D^-1 L, GEMMs for X, Rd, Ld, Dd
 * (solver.py:224-262); status / rcond / outputs exactly as skel_factor_level.
 * dd_off .. lam_off: the box's output offsets; work: skel_factor_big_bytes. */
int64_t skel_factor_big_bytes(int32_t n, int32_t k, int32_t field);
int skel_factor_big(const SkelFactorLevel* F, int32_t box, int32_t n, int32_t k, int64_t dd_off,
                    int64_t ld_off, int64_t rd_off, int64_t lam_off, void* work, int64_t work_bytes,
                    int32_t field, void* stream);
int skel_dense_inverse_big(void* A, int32_t n, double regularize, int32_t* status, int32_t field,
                           void* scratch, void* stream);

/* ---- multi-RHS solve / apply sweeps (solver.py:279-318, skel.py:206-249) */

/* out[koff[a]+t, :] = sum_j M_a[t, j] u[noff[a]+j, :]   (M_a: k x n row-major
 * at m_off[a]); vectors row-major with R values per row.  max_n / max_k bound
 * n and k over the processed boxes: order[0..nbox) when order != NULL (a
 * size bucket), else boxes 0..nbox-1.
 * Up-sweep of solve (solver.py:295-302) / apply (skel.py:225-232). */
int skel_sweep_up_ex(int32_t nbox, const int32_t* n, const int32_t* k,
                     const int64_t* noff, const int64_t* koff, const int64_t* m_off,
                     const void* M, const void* u, void* out, int32_t R, int32_t field,
                     int32_t max_n, int32_t max_k, const int32_t* order, void* stream);

/* w[noff[a]+i, :] = sum_j A_a[i,j] u[noff[a]+j, :] + sum_t B_a[i,t] v[koff[a]+t, :]
 * (A_a: n x n at a_off[a], B_a: n x k at b_off[a], row-major); max_n / max_k
 * bound n and k.  Down-sweep of solve (solver.py:304-314) / apply (skel.py:235-244). */
int skel_sweep_down_ex(int32_t nbox, const int32_t* n, const int32_t* k,
                       const int64_t* noff, const int64_t* koff, const int64_t* a_off,
                       const void* A, const int64_t* b_off, const void* B,
                       const void* u, const void* v, void* w, int32_t R, int32_t field,
                       int32_t max_n, int32_t max_k, const int32_t* order, void* stream);

/* The same sweeps with the finest level's tree-order gather / scatter of the
 * right-hand sides fused in (solver.py:288,316-318): u rows are read as
 * u[urows[noff[a] + j]] and w rows written to w[wrows[noff[a] + i]] (NULL =
 * plain).  R <= 16 (returns -3 otherwise). */
int skel_sweep_up_rows(int32_t nbox, const int32_t* n, const int32_t* k, const int64_t* noff,
                       const int64_t* koff, const int64_t* m_off, const void* M, const void* u,
                       void* out, int32_t R, int32_t field, int32_t max_n, int32_t max_k,
                       const int32_t* order, const int64_t* urows, void* stream);
int skel_sweep_down_rows(int32_t nbox, const int32_t* n, const int32_t* k, const int64_t* noff,
                         const int64_t* koff, const int64_t* a_off, const void* A,
                         const int64_t* b_off, const void* B, const void* u, const void* v, void* w,
                         int32_t R, int32_t field, int32_t max_n, int32_t max_k,
                         const int32_t* order, const int64_t* urows, const int64_t* wrows,
                         void* stream);

/* y = M x for a dense K x K row-major M, R columns (top-level S^-1 / S). */
int skel_dense_apply(const void* M, int32_t K, int32_t Kc, const void* x, void* y,
                     int32_t R, int32_t field, void* stream);

/* Row gather / scatter by the tree permutation: dst[i,:] = src[perm[i],:]
 * (gather) or dst[perm[i],:] = src[i,:] (scatter), N x R. */
int skel_permute_rows(const int64_t* perm, int64_t N, const void* src, void* dst,
                      int32_t R, int32_t scatter, int32_t field, void* stream);

/* Segment compaction: dst[dst_off[b] + t] = src[src_off[b] + t], t < len[b]. */
int skel_compact_i32(int32_t nseg, const int64_t* src_off, const int32_t* len,
                     const int64_t* dst_off, const int32_t* src, int32_t* dst,
                     void* stream);

/* On-the-fly dense matvec y = A x with exact entries (bie.py:174-176 without
 * materialising A), x/y in TREE order, R columns. */
int skel_dense_matvec(const SkelSource* src, const void* x, void* y, int32_t R,
                      int32_t field, void* stream);

/* ---- host-side tree + neighbour lists (geom.py:118-219), native C++ ----- */

/* Build the adaptive orthtree (geom.py:118-184). Returns an opaque handle. */
int skel_tree_build(const double* coords, int64_t n, int32_t dim, int64_t max_leaf,
                    void** handle);
/* Node / cover counts. */
int skel_tree_sizes(void* handle, int64_t* nnodes, int32_t* ncovers);
/* Copy out node arrays (nnodes each; center nnodes*dim) and perm (n). */
int skel_tree_nodes(void* handle, double* center, double* hw, int64_t* lo, int64_t* hi,
                    int64_t* depth, int64_t* parent, int64_t* nchild, int64_t* perm);
/* Cover li (0 = finest): number of boxes, and ids if out != NULL. */
int skel_tree_cover(void* handle, int32_t li, int64_t* count, int64_t* ids);
/* Same-cover adjacency (geom.py:205-219), O(p) grid hash; CSR. count gets
 * the number of adjacency entries; pass idx = NULL to query it. */
int skel_tree_neighbors(void* handle, int32_t li, int64_t* off, int64_t* count,
                        int64_t* idx);
/* Borrowed pointer to the tree permutation (n int64, tree position -> original
 * index; read-only, valid until skel_tree_free): lets the caller wrap it without
 * the 8 n-byte copy skel_tree_nodes makes when given a perm buffer. */
int skel_tree_perm_ptr(void* handle, const int64_t** perm);
int skel_tree_free(void* handle);
/* PointSet validation (geom.py:42 and the unit-normal rule): 0 ok, -3 a
 * non-finite coordinate, -4 a normal with | |n| - 1 | > 1e-12 (normals may be
 * NULL); |n| is formed as np.linalg.norm(axis=1) does. */
int skel_check_points(const double* coords, const double* normals, int64_t n, int32_t dim);
/* mean(w[perm]) with numpy's float64 pairwise summation order (bit-identical
 * to np.mean(w[perm])): the proxy weight scale of _BieSource (bie.py:251). */
int skel_perm_mean(const double* w, const int64_t* perm, int64_t n, double* out);

/* FP64 throughput probe: kind 0 = DFMA chains, 1 = DMMA (mma.sync m8n8k4
 * f64).  *flops receives the launch's flop count; time it with events. */
int skel_fp64_probe(int32_t kind, int32_t iters, double* scratch, double* flops,
                    void* stream);

/* Library self-description (for the loader's symbol check). */
const char* skel_version(void);
int skel_device_query(int32_t* sm_count, int32_t* smem_optin, int32_t* cc_major,
                      int32_t* cc_minor);

#ifdef __cplusplus
}
#endif
#endif /* SKEL_B200_H */
