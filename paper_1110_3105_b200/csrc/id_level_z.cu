// id_level_z.cu -- complex128 instantiations of the level ID kernels
// (id_level.cuh), split from id_level.cu so the two compile in parallel.
#include "id_level.cuh"

int id_level_zc(const SkelSource* src, const SkelLevel* lv, const int32_t* order, int nrun,
                int max_m, int max_n, int64_t max_w, cudaStream_t st) {
  return id_level_impl<zc>(src, lv, order, nrun, max_m, max_n, max_w, st);
}

int id_batched_zc(const void* A, const int64_t* a_off, const int32_t* m, const int32_t* n, int nmat,
                  double eps, const int32_t* min_rank, int32_t* rank, int32_t* skel,
                  const int64_t* skel_off, void* proj, const int64_t* proj_off, double* bigP,
                  double* ratio, void* scratch, int64_t scratch_bytes, int max_m, int max_n,
                  cudaStream_t st, void* rfac, const int64_t* rfac_off) {
  return id_batched_impl<zc>(A, a_off, m, n, nmat, eps, min_rank, rank, skel, skel_off, proj,
                             proj_off, bigP, ratio, scratch, scratch_bytes, max_m, max_n, st, rfac,
                             rfac_off);
}
