// id_level.cu -- C-ABI entry points of the K1 + K2 level kernels (templates
// in id_level.cuh; the complex instantiations are compiled in id_level_z.cu).
#include "id_level.cuh"

extern "C" {

int skel_id_level(const SkelSource* src, const SkelLevel* lv, const int32_t* box_order,
                  int32_t nbox_run, int32_t max_m, int32_t max_n, int64_t max_w, int32_t field,
                  void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (field == 0) return id_level_impl<double>(src, lv, box_order, nbox_run, max_m, max_n, max_w, st);
  return id_level_zc(src, lv, box_order, nbox_run, max_m, max_n, max_w, st);
}

int skel_assemble_D(const SkelSource* src, const SkelLevel* lv, const int32_t* order, int32_t nrun,
                    int32_t max_n, int32_t field, void* stream) {
  const int nb = order ? nrun : lv->nbox;
  if (nb <= 0) return 0;
  if (max_n < 1) max_n = 1;
  cudaStream_t st = (cudaStream_t)stream;
  const int chunk = max_n < 512 ? max_n : 512;
  size_t smem = sizeof(Pt) * (size_t)chunk;
  // few big boxes (3D coarse levels): split each box's rows over CTAs
  const int sms = skel_sm_count();
  int gy = 1;
  if (nb < 2 * sms && max_n > 64) {
    gy = (2 * sms + nb - 1) / nb;
    const int cap = (max_n + 31) / 32;
    if (gy > cap) gy = cap;
  }
  dim3 grid(nb, gy);
  if (field == 0) {
    SKEL_TRY(cudaFuncSetAttribute(k_assemble_D<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_assemble_D<double><<<grid, 128, smem, st>>>(*src, *lv, chunk, order);
  } else {
    SKEL_TRY(cudaFuncSetAttribute(k_assemble_D<zc>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_assemble_D<zc><<<grid, 128, smem, st>>>(*src, *lv, chunk, order);
  }
  return skel_last_error();
}

int skel_id_batched(const void* A, const int64_t* a_off, const int32_t* m, const int32_t* n,
                    int32_t nmat, double eps, const int32_t* min_rank, int32_t* rank,
                    int32_t* skel, const int64_t* skel_off, void* proj, const int64_t* proj_off,
                    double* bigP, double* ratio, int32_t field, void* scratch, int64_t scratch_bytes,
                    int32_t max_m, int32_t max_n, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (field == 0)
    return id_batched_impl<double>(A, a_off, m, n, nmat, eps, min_rank, rank, skel, skel_off, proj,
                                   proj_off, bigP, ratio, scratch, scratch_bytes, max_m, max_n, st);
  return id_batched_zc(A, a_off, m, n, nmat, eps, min_rank, rank, skel, skel_off, proj,
                       proj_off, bigP, ratio, scratch, scratch_bytes, max_m, max_n, st);
}

int skel_pivoted_qr_batched(const void* A, const int64_t* a_off, const int32_t* m, const int32_t* n,
                            int32_t nmat, double eps, const int32_t* min_rank, int32_t* rank,
                            int32_t* piv, const int64_t* piv_off, void* rfac, const int64_t* rfac_off,
                            void* proj, const int64_t* proj_off, double* bigP, double* ratio,
                            int32_t field, void* scratch, int64_t scratch_bytes, int32_t max_m,
                            int32_t max_n, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!rfac || !rfac_off) return -1;
  if (field == 0)
    return id_batched_impl<double>(A, a_off, m, n, nmat, eps, min_rank, rank, piv, piv_off, proj,
                                   proj_off, bigP, ratio, scratch, scratch_bytes, max_m, max_n, st,
                                   rfac, rfac_off);
  return id_batched_zc(A, a_off, m, n, nmat, eps, min_rank, rank, piv, piv_off, proj, proj_off,
                       bigP, ratio, scratch, scratch_bytes, max_m, max_n, st, rfac, rfac_off);
}

int skel_assemble_S(const SkelSource* src, const int32_t* rows, const int32_t* rbox, int32_t Kr,
                    const int32_t* cols, const int32_t* cbox, int32_t Kc, void* S, int32_t field,
                    void* stream) {
  int64_t tot = (int64_t)Kr * Kc;
  if (tot == 0) return 0;
  int blocks = (int)((tot + 255) / 256);
  cudaStream_t st = (cudaStream_t)stream;
  if (field == 0) k_assemble_S<double><<<blocks, 256, 0, st>>>(*src, rows, rbox, Kr, cols, cbox, Kc, (double*)S);
  else k_assemble_S<zc><<<blocks, 256, 0, st>>>(*src, rows, rbox, Kr, cols, cbox, Kc, (zc*)S);
  return skel_last_error();
}

int skel_eval_block(const SkelSource* src, const int32_t* rows, int32_t m, const int32_t* cols,
                    int32_t n, void* out, int32_t field, void* stream) {
  int64_t tot = (int64_t)m * n;
  if (tot == 0) return 0;
  int blocks = (int)((tot + 255) / 256);
  cudaStream_t st = (cudaStream_t)stream;
  if (field == 0) k_eval_block<double><<<blocks, 256, 0, st>>>(*src, rows, m, cols, n, (double*)out);
  else k_eval_block<zc><<<blocks, 256, 0, st>>>(*src, rows, m, cols, n, (zc*)out);
  return skel_last_error();
}

int skel_dense_matvec(const SkelSource* src, const void* x, void* y, int32_t R, int32_t field,
                      void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int blocks = (int)((src->n + 255) / 256);
  for (int c0 = 0; c0 < R; c0 += 4) {
    if (field == 0) {
      if (R == 1) k_dense_matvec<double, 1><<<blocks, 256, 0, st>>>(*src, (const double*)x, (double*)y, R, c0);
      else k_dense_matvec<double, 4><<<blocks, 256, 0, st>>>(*src, (const double*)x, (double*)y, R, c0);
    } else {
      if (R == 1) k_dense_matvec<zc, 1><<<blocks, 256, 0, st>>>(*src, (const zc*)x, (zc*)y, R, c0);
      else k_dense_matvec<zc, 4><<<blocks, 256, 0, st>>>(*src, (const zc*)x, (zc*)y, R, c0);
    }
    SKEL_TRY(cudaGetLastError());
  }
  return 0;
}

}  // extern "C"
